#!/bin/bash
# A/B of library builds over several configs (kernel-only): ab_libs.sh "<cfgs>" lib1.so lib2.so ...
cfgs="$1"; shift
for lib in "$@"; do echo "== $lib"; XDROP_LIB=$lib CFGS="$cfgs" python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2309_07270_b200 as xd
from synth import workload as W
for name in os.environ["CFGS"].split():
    nm, _, x = name.partition(":")
    w = W.config("celegans", scale=0.05) if nm == "celegans" else W.config(nm)
    X = int(x) if x else w.X
    with xd.Aligner() as al:
        ts = []
        for _ in range(3):
            r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
            st = al.stats(); ts.append(st["total_ms"])
    print(f"  {name:12s} total_ms={min(ts):8.2f} GCUPS={c.sum()/min(ts)/1e6:7.1f} lvl={['%.1f'%t for t in st['level_ms']]} esc={st['escalated'][:4]} score_sum={int(r['score'].sum())} cells={int(c.sum())}", flush=True)
PY
done
