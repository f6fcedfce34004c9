"""Scratch: lane-mode warp efficiency estimate (sum of per-extension anti-diagonals vs 32 x batch max)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config(sys.argv[1] if len(sys.argv) > 1 else "ecoli")
with xd.Aligner() as al:
    r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    st = al.stats()
p = w.pairs.reshape(-1, 4).astype(np.int64)
lens = np.diff(w.offsets)
la, lb = lens[p[:, 0]], lens[p[:, 1] & 0x7fffffff]
k = w.k
wl = np.minimum(p[:, 2], p[:, 3]); wr = np.minimum(la - p[:, 2] - k, lb - p[:, 3] - k)
dl = (p[:, 2] - r["a_begin"]) + (p[:, 3] - r["b_begin"])
dr = (r["a_end"] - p[:, 2] - k) + (r["b_end"] - p[:, 3] - k)
cost = np.empty(2 * len(p), np.int64); cost[0::2] = wl; cost[1::2] = wr
dd = np.empty(2 * len(p), np.int64); dd[0::2] = dl; dd[1::2] = dr
dd += 2 * w.X   # X-drop overshoot (rough)
order = np.argsort(-(cost >> 4), kind="stable")
nl = st["long_items"]
o = order[nl:]
n = len(o) // 32 * 32
B = dd[o[:n]].reshape(-1, 32)
eff = B.sum() / (32 * B.max(1).sum())
print(f"items {len(dd)} long {nl} lane batches {len(B)} warp efficiency {eff:.3f}")
print(f"cost vs actual: corr {np.corrcoef(cost, dd)[0,1]:.3f}; frac actual < cost/4: {(dd < cost/4).mean():.3f}")
# if sorted by actual length (oracle order): upper bound
B2 = np.sort(dd[o])[::-1][:n].reshape(-1, 32)
print(f"efficiency if batches were sorted by actual length: {B2.sum() / (32 * B2.max(1).sum()):.3f}")
