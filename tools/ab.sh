#!/bin/bash
# A/B of library builds on the E. coli-shaped batch (kernel-only timing)
for lib in "$@"; do echo "== $lib"; XDROP_LIB=$lib XDROP_LONG_G=4 XDROP_LONG_ALPHA=1.0 python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
with xd.Aligner() as al:
    ts = []
    for _ in range(4):
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        ts.append(al.stats()["level_ms"][0])
print(f"kernel_ms={min(ts):.2f} GCUPS={c.sum()/min(ts)/1e6:.1f} all={['%.2f'%t for t in ts]}")
PY
done
