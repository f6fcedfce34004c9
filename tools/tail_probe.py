"""Scratch experiment: how much of the band kernel is the critical path of the longest extensions?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W

w = W.config("ecoli")
lens = np.diff(w.offsets)
p = w.pairs
estL = np.minimum(p[:, 2], p[:, 3])
estR = np.minimum(lens[p[:, 0]] - p[:, 2], lens[p[:, 1]] - p[:, 3]) - w.k
est = np.maximum(estL, estR)
order = np.argsort(-est)
al = xd.Aligner()
def run(idx, tag):
    sub = p[np.sort(idx)]
    for _ in range(2):
        r, c = al.align(w.seq, w.offsets, sub, k=w.k, X=w.X)
    st = al.stats()
    print(f"{tag:28s} pairs={len(idx):6d} cells={c.sum():.3e} kernel_ms={st['level_ms'][0]:.2f} "
          f"GCUPS={c.sum()/st['level_ms'][0]/1e6:.1f} max_est={est[idx].max()} esc={st['escalated'][:3]}")
run(order, "full")
for f in [0.005, 0.02, 0.1]:
    k = int(len(order) * f)
    run(order[k:], f"without top {f*100:.1f}%")
    run(order[:k], f"only top {f*100:.1f}%")
run(order[len(order)//2:], "shorter half")
