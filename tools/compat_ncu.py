"""One E. coli-shaped call in the default mode, then one in the compat mode (for an ncu comparison of
pk_tiered_kernel<4,8,false> vs <4,8,true>; profiles/compat_r2.md)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd
from synth import workload as W
w = W.config("ecoli")
for compat in (False, True):
    with xd.Aligner(seqan_compat=compat) as al:
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        print("compat" if compat else "default", int(c.sum()), al.stats()["kernel_ms"], flush=True)
