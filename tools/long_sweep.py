"""Scratch experiment: long-extension mode (lanes per extension, cut alpha) vs kernel time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W

w = W.config(sys.argv[1] if len(sys.argv) > 1 else "ecoli")
ref = None
for g, a in [(0, 0.5), (2, 0.3), (2, 0.5), (2, 1.0), (4, 0.3), (4, 0.5), (4, 1.0), (4, 2.0)]:
    os.environ["XDROP_LONG_G"], os.environ["XDROP_LONG_ALPHA"] = str(g), str(a)
    with xd.Aligner() as al:
        ts = []
        for _ in range(3):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            ts.append(al.stats()["level_ms"][0])
        st = al.stats()
    if ref is None:
        ref = (r, c)
    same = np.array_equal(r, ref[0]) and np.array_equal(c, ref[1])
    print(f"G={g} alpha={a:4.1f} long={st['long_items']:6d} kernel_ms={min(ts):7.2f} "
          f"GCUPS={c.sum()/min(ts)/1e6:7.1f} esc={st['escalated'][:3]} same={same}", flush=True)
