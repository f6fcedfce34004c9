#!/bin/bash
# A/B of env settings on the same library (E. coli-shaped; kernel-only): ab_env.sh "XDROP_PK16=0" "XDROP_PK16=1" ...
for cfg in "$@"; do echo "== $cfg"; env $cfg python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
with xd.Aligner() as al:
    ts = []
    for _ in range(4):
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats(); ts.append(st["level_ms"][0])
print(f"kernel_ms={min(ts):.2f} GCUPS={c.sum()/min(ts)/1e6:.1f} esc={st['escalated'][:3]} lvl_items={st['level_items']} all={['%.2f'%t for t in ts]} score_sum={int(r['score'].sum())}")
PY
done
