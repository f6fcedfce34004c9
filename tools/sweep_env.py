"""Scratch: kernel time of one config under several env settings (each a fresh context; the env is
read by xdrop_init).  python tools/sweep_env.py <cfg>[:X] "K=V K2=V2" "K=V" ...   (cfg celegans = x0.05)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
nm, _, x = sys.argv[1].partition(":")
w = W.config("celegans", scale=0.05) if nm == "celegans" else W.config(nm)
if x:
    w = w.with_X(int(x))
ref = None
base_env = dict(os.environ)
for setting in sys.argv[2:]:
    os.environ.clear(); os.environ.update(base_env)
    for kv in setting.split():
        k, v = kv.split("=")
        os.environ[k] = v
    with xd.Aligner() as al:
        ts, ks = [], []
        for _ in range(3):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            st = al.stats(); ts.append(st["kernel_ms"]); ks.append(st["band_kernel"])
    if ref is None:
        ref = (r, c)
    same = np.array_equal(r, ref[0]) and np.array_equal(c, ref[1])
    print(f"{nm}:{w.X} [{setting}] kernel_ms={min(ts):7.2f} all={['%.1f' % t for t in ts]} kern={ks} "
          f"GCUPS={c.sum() / min(ts) / 1e6:7.1f} long={st['long_items']} esc={st['escalated'][:3]} "
          f"lvl_ms={['%.1f' % t for t in st['level_ms']]} same={same}", flush=True)
