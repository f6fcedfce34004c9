"""Scratch: where does the band kernel's time go?  Work-unit timeline (XDROP_TIMELINE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["XDROP_TIMELINE"] = "1"
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config(sys.argv[1] if len(sys.argv) > 1 else "ecoli")
with xd.Aligner() as al:
    for _ in range(2):
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    tl = al.timeline(); st = al.stats()
t0 = tl[:, 2].min(); T = (tl[:, 3].max() - t0) / 1e6
print(f"kernel span {T:.2f} ms, units {len(tl)}, stolen {st['stolen']}, band ms {st['level_ms'][0]:.2f}")
names = ["lane", "long", "stolen", "pair", "warp", "endgame"]
for ty in range(6):
    m = tl[:, 0] == ty
    if m.any():
        d = (tl[m, 3] - tl[m, 2]) / 1e6
        print(f"  {names[ty]:6s} n={m.sum():6d} dur mean {d.mean():.2f} max {d.max():.2f} ms; "
              f"last end {(tl[m, 3].max() - t0) / 1e6:.2f} ms, last start {(tl[m, 2].max() - t0) / 1e6:.2f} ms")
# busy warps over time
nw = tl[:, 1].max() + 1
edges = np.linspace(0, T, 21)
for a, b in zip(edges[:-1], edges[1:]):
    lo, hi = t0 + a * 1e6, t0 + b * 1e6
    busy = ((np.minimum(tl[:, 3], hi) - np.maximum(tl[:, 2], lo)).clip(0)).sum() / ((hi - lo) * nw)
    print(f"  [{a:5.1f},{b:5.1f}) ms busy warps {busy*100:5.1f}%")
