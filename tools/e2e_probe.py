"""Scratch: where the host-API (e2e) call's time goes beyond the device pipeline."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
seq_h = torch.from_numpy(w.seq).pin_memory().numpy()
off_h = torch.from_numpy(w.offsets).pin_memory().numpy()
pairs_h = torch.from_numpy(w.pairs).pin_memory().numpy()
with xd.Aligner() as al:
    for i in range(4):
        t0 = time.perf_counter()
        r, c = al.align(seq_h, off_h, pairs_h, k=w.k, X=w.X)
        t1 = time.perf_counter()
        st = al.stats(); ss = al.sched_stats()
        print(f"wall {1e3*(t1-t0):.2f} ms  lib span {ss['span_ms']:.2f}  device total {st['total_ms']:.2f} pack {st['pack_ms']:.2f} kernel {st['kernel_ms']:.2f}")
    a = torch.empty(w.seq.nbytes, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(seq_h)
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        a.copy_(src, non_blocking=True); torch.cuda.synchronize()
        print(f"H2D {w.seq.nbytes/1e6:.0f} MB pinned: {1e3*(time.perf_counter()-t0):.2f} ms")
    t0 = time.perf_counter(); out = np.zeros(w.n_pairs, dtype=xd.RESULT_DTYPE); cc = np.zeros(w.n_pairs, np.int64); print(f"np.zeros {1e3*(time.perf_counter()-t0):.3f} ms")
