import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.random_pairs_workload(seed=19, n_pairs=3, len_lo=4500, len_hi=5000, k=5, X=100000, related=0.0)
with xd.Aligner() as al:
    r, c = al.align(w.seq, w.offsets, w.pairs, k=5, X=100000)
    print(r, c, al.stats()["escalated"])
