import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
for X in (50, 100):
    w = W.config("xsweep").with_X(X)
    with xd.Aligner() as al:
        for _ in range(2):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
            st = al.stats()
            print(X, st["band_kernel"], st["escalated"], "cta", st["cta_items"], st["level_ms"], st["level_items"])
