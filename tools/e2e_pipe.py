import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
seq_h = torch.from_numpy(w.seq).pin_memory().numpy()
off_h = torch.from_numpy(w.offsets).pin_memory().numpy()
pairs_h = torch.from_numpy(w.pairs).pin_memory().numpy()
K = 12
for nctx in (1, 2, 3):
    als = [xd.Aligner() for _ in range(nctx)]
    for al in als:
        al.align(seq_h, off_h, pairs_h, k=w.k, X=w.X)
    cells = [0] * nctx
    def run(i):
        c = 0
        for s in range(i, K, nctx):
            r, cc = als[i].align(seq_h, off_h, pairs_h, k=w.k, X=w.X)
            c += int(cc.sum())
        cells[i] = c
    t0 = time.perf_counter()
    th = [threading.Thread(target=run, args=(i,)) for i in range(nctx)]
    for t in th: t.start()
    for t in th: t.join()
    dt = time.perf_counter() - t0
    print(f"contexts={nctx}: {K} batches in {dt*1e3:.1f} ms = {dt*1e3/K:.2f} ms/batch, {sum(cells)/dt/1e9:.0f} GCUPS", flush=True)
    for al in als: al.close()
