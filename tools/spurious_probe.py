"""Scratch: the X-sweep's spurious extensions alone -- kernel time of N of them (lowest scores of the
full batch) under each packed kernel and env setting, i.e. the per-anti-diagonal chain latency of the
shapes they run in when the GPU is otherwise idle.  python tools/spurious_probe.py [N] ["K=V ..."]..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("xsweep")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
with xd.Aligner() as al:
    r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
sub = w.pairs[np.argsort(r["score"])[:N]]
lens = np.diff(w.offsets)
base_env = dict(os.environ)
for setting in (sys.argv[2:] or [""]):
    os.environ.clear(); os.environ.update(base_env)
    for kv in setting.split():
        k, v = kv.split("="); os.environ[k] = v
    for kernel in ("tiered", "shared"):
        with xd.Aligner(kernel=kernel) as al:
            ts = []
            for _ in range(3):
                rr, cc = al.align(w.seq, w.offsets, sub, k=w.k, X=w.X)
                st = al.stats(); ts.append(st["kernel_ms"])
        ad = 2 * int(lens[sub[:, 0]].max())
        print(f"[{setting}] {kernel:6s} N={N} kernel_ms={min(ts):7.2f} cells={cc.sum():.3e} "
              f"esc={st['escalated']} endsteal={st.get('endgame_stolen')} "
              f"~ns/antidiag(longest {ad})={min(ts) * 1e6 / ad:.0f}", flush=True)
