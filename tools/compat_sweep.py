"""Scratch: compat-mode kernel time per config under env settings (XDROP_COMPAT_GRP: the probe
fraction above which the warp-ring kernel takes the batch first).  python tools/compat_sweep.py "K=V" ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
cfgs = [("ecoli", 1.0, 15), ("ecoli", 0.05, 15), ("xsweep", 1.0, 15), ("xsweep", 1.0, 50), ("celegans", 0.05, 15)]
base = dict(os.environ)
for setting in sys.argv[1:] or [""]:
    os.environ.clear(); os.environ.update(base)
    for kv in setting.split():
        k, v = kv.split("="); os.environ[k] = v
    for name, scale, X in cfgs:
        w = W.config(name, scale=scale).with_X(X)
        with xd.Aligner(seqan_compat=True) as al:
            ts = []
            for _ in range(2):
                r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
                st = al.stats(); ts.append(st["kernel_ms"])
        print(f"[{setting}] {name} x{scale} X={X}: {min(ts):7.1f} ms {c.sum() / min(ts) / 1e6:6.0f} GCUPS "
              f"probe={st['probe_overflows']} esc={st['escalated']}", flush=True)
