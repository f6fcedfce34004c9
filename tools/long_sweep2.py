import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
for g, a in [(4, 1.0), (4, 0.85), (4, 0.7), (2, 0.85), (2, 0.7), (2, 0.6), (4, 1.2), (0, 1.0)]:
    os.environ["XDROP_LONG_G"], os.environ["XDROP_LONG_ALPHA"] = str(g), str(a)
    with xd.Aligner() as al:
        ts = []
        for _ in range(4):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            ts.append(al.stats()["level_ms"][0])
        st = al.stats()
    print(f"G={g} alpha={a:4.2f} long={st['long_items']:6d} kernel_ms={min(ts):7.2f} GCUPS={c.sum()/min(ts)/1e6:7.1f} all={['%.2f'%t for t in ts]}", flush=True)
