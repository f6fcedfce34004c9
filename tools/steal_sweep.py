import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config(sys.argv[1] if len(sys.argv) > 1 else "ecoli")
for sm in ["0", "512", "1024", "2048", "4096"]:
    os.environ["XDROP_STEAL_MIN"] = sm
    with xd.Aligner() as al:
        ts = []
        for _ in range(4):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            ts.append(al.stats()["level_ms"][0])
        st = al.stats()
    print(f"steal_min={sm:5s} stolen={st['stolen']:6d} kernel_ms={min(ts):7.2f} GCUPS={c.sum()/min(ts)/1e6:7.1f} all={['%.2f'%t for t in ts]}", flush=True)
