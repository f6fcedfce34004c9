"""Throughput of the SeqAn/LOGAN-style compat mode (XDROP_FLAG_SEQAN_COMPAT) next to the default mode
on the BASELINE configs 2 and 4 shapes, with an oracle check of a sample of every batch
(-> profiles/compat_r2.md).  python tools/compat_bench.py [out.md]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
import paper_2309_07270_b200 as xd
from synth import workload as W

rows = []
for name, X in [("ecoli", 15), ("xsweep", 15), ("xsweep", 50), ("xsweep", 100)]:
    w = W.config(name).with_X(X)
    line = [f"{name} X={X}", f"{w.n_pairs:,}"]
    for compat in (False, True):
        with xd.Aligner(seqan_compat=compat) as al:
            ts = []
            for _ in range(2):
                res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
                st = al.stats()
                ts.append(st["kernel_ms"])
        ms = min(ts)
        line += [f"{ms:.1f}", f"{cells.sum() / ms / 1e6:.0f}"]
        if compat:
            idx = np.arange(0, w.n_pairs, max(1, w.n_pairs // 400))
            ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs[idx], w.k, X=X, compat=True)
            ok = all((res[f][idx] == ref[f]).all() for f in ("score", "a_begin", "a_end", "b_begin", "b_end"))
            ok = ok and (cells[idx] == rc).all()
            line += [f"{st['escalated'][2]} / {st['escalated'][3]}",
                     "[" + ", ".join(f"{t:.1f}" for t in st["level_ms"]) + "]",
                     f"{idx.size} pairs {'bit-exact' if ok else 'MISMATCH'}"]
    rows.append(line)
    print(" | ".join(line), flush=True)

out = sys.argv[1] if len(sys.argv) > 1 else None
if out:
    with open(out, "w") as f:
        f.write("# Compat mode (XDROP_FLAG_SEQAN_COMPAT) vs default mode, 1 x B200\n\n")
        f.write("`python tools/compat_bench.py`: kernel time (ms, best of 2) and GCUPS (each mode's own DP cells) "
                "of the default packed path and of the compat mode's general-path kernels; ring overflows = "
                "extensions redone by the 8-warp ring / the global-memory kernel; level_ms = [ring kernels, -, -, "
                "global-memory kernel]; every batch's sample checked against the oracle's compat mode.\n\n")
        f.write("| batch | pairs | default ms | default GCUPS | compat ms | compat GCUPS | ring overflows | "
                "level_ms | oracle sample |\n|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write("| " + " | ".join(r) + " |\n")
