import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config(sys.argv[1] if len(sys.argv) > 1 else "ecoli")
for eg in ["0", "0.1", "0.25", "0.5", "1.0"]:
    os.environ["XDROP_ENDGAME"] = eg
    with xd.Aligner() as al:
        ts = []
        for _ in range(4):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            ts.append(al.stats()["level_ms"][0])
    print(f"endgame={eg:5s} kernel_ms={min(ts):7.2f} GCUPS={c.sum()/min(ts)/1e6:7.1f} all={['%.2f'%t for t in ts]}", flush=True)
