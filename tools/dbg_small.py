import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
import oracle
w = W.random_pairs_workload(seed=1, n_pairs=50, len_lo=30, len_hi=300, k=11, X=15)
with xd.Aligner() as al:
    r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, M=1, mu=-1, g=-1, X=15)
bad = np.nonzero((r['score'] != ref['score']) | (c != rc))[0]
print(os.environ.get("XDROP_LIB"), "bad", len(bad), "of", len(r))
for i in bad[:5]:
    print(w.pairs[i], r[i], ref[i], c[i], rc[i])
