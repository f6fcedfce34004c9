"""Scratch: the 500 longest E. coli-shaped pairs alone (one warp per scheduler or less)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
lens = np.diff(w.offsets); p = w.pairs
est = np.maximum(np.minimum(p[:, 2], p[:, 3]), np.minimum(lens[p[:, 0]] - p[:, 2], lens[p[:, 1]] - p[:, 3]) - w.k)
sub = p[np.argsort(-est)[:int(os.environ.get("NPAIRS", "500"))]]
with xd.Aligner() as al:
    for _ in range(int(os.environ.get("REPS", "2"))):
        r, c = al.align(w.seq, w.offsets, sub, k=w.k, X=w.X)
        st = al.stats()
        print(f"pairs={len(sub)} kernel_ms={st['level_ms'][0]:.2f} cells={c.sum():.3e} long={st['long_items']}")
