"""Scratch: run one config through the host API (for ncu captures): run_cfg.py <name>[:X] [reps]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
nm, _, x = sys.argv[1].partition(":")
w = W.config("celegans", scale=0.05) if nm == "celegans" else W.config(nm)
X = int(x) if x else w.X
with xd.Aligner() as al:
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
        print(al.stats()["level_ms"], flush=True)
