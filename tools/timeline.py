"""Scratch: where does the band kernel's time go?  Work-unit timeline (XDROP_TIMELINE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["XDROP_TIMELINE"] = "1"
import numpy as np
import paper_2309_07270_b200 as xd
from synth import workload as W
_nm, _, _x = (sys.argv[1] if len(sys.argv) > 1 else "ecoli").partition(":")
w = W.config(_nm, scale=0.05) if _nm == "celegans" else W.config(_nm)
if os.environ.get("TL_KERNEL"):
    os.environ["XDROP_KERNEL"] = os.environ["TL_KERNEL"]
if _x:
    w = w.with_X(int(_x))
with xd.Aligner() as al:
    for _ in range(2):
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    print(al.stats()['band_kernel'], al.stats()['level_ms'])
    tl = al.timeline(); st = al.stats()
t0 = tl[:, 2].min(); T = (tl[:, 3].max() - t0) / 1e6
print(f"kernel span {T:.2f} ms, units {len(tl)}, stolen {st['stolen']}, band ms {st['level_ms'][0]:.2f}")
names = ["lane", "long", "stolen", "pair", "warp", "endgame", "t3", "endsteal"]
for ty in range(8):
    m = tl[:, 0] == ty
    if m.any():
        d = (tl[m, 3] - tl[m, 2]) / 1e6
        print(f"  {names[ty]:6s} n={m.sum():6d} warp-ms {d.sum():9.1f} dur mean {d.mean():.2f} max {d.max():.2f} ms; "
              f"last end {(tl[m, 3].max() - t0) / 1e6:.2f} ms, last start {(tl[m, 2].max() - t0) / 1e6:.2f} ms")
# busy warps over time
nw = tl[:, 1].max() + 1
edges = np.linspace(0, T, 21)
for a, b in zip(edges[:-1], edges[1:]):
    lo, hi = t0 + a * 1e6, t0 + b * 1e6
    busy = ((np.minimum(tl[:, 3], hi) - np.maximum(tl[:, 2], lo)).clip(0)).sum() / ((hi - lo) * nw)
    per = []
    for ty in range(8):
        m = tl[:, 0] == ty
        if m.any():
            bt = ((np.minimum(tl[m, 3], hi) - np.maximum(tl[m, 2], lo)).clip(0)).sum() / ((hi - lo) * nw)
            if bt > 0.005:
                per.append(f"{names[ty]} {bt*100:4.1f}")
    print(f"  [{a:5.1f},{b:5.1f}) ms busy warps {busy*100:5.1f}%   " + ", ".join(per))
# the latest-ending work units
if len(sys.argv) > 2:
    o = np.argsort(-tl[:, 3])[:int(sys.argv[2])]
    for i in o:
        print(f"  late: {names[tl[i,0]]:6s} start {(tl[i,2]-t0)/1e6:6.2f} end {(tl[i,3]-t0)/1e6:6.2f} ms")
    for ty in (0,):
        m = tl[:, 0] == ty
        d = (tl[m, 3] - tl[m, 2]) / 1e6; s = (tl[m, 2] - t0) / 1e6
        for a in range(0, 16, 2):
            mm = (s >= a) & (s < a + 2)
            if mm.any(): print(f"  lane units starting [{a},{a+2}) ms: n={mm.sum()} dur mean {d[mm].mean():.2f} max {d[mm].max():.2f}")
# start-up: units started and warps busy per 0.1 ms over the first 2.5 ms
if os.environ.get("TL_START"):
    for a in np.arange(0, 2.5, 0.1):
        lo, hi = t0 + a * 1e6, t0 + (a + 0.1) * 1e6
        st_n = ((tl[:, 2] >= lo) & (tl[:, 2] < hi))
        busy = ((np.minimum(tl[:, 3], hi) - np.maximum(tl[:, 2], lo)).clip(0)).sum() / ((hi - lo) * nw)
        kinds = np.bincount(tl[st_n, 0], minlength=8)
        print(f"  [{a:4.1f},{a+0.1:4.1f}) started {st_n.sum():5d} by kind {kinds.tolist()} busy {busy*100:5.1f}%")
if os.environ.get("TL_START"):
    for ty in range(8):
        m = (tl[:, 0] == ty) & (tl[:, 2] - t0 < 2.5e6)
        if m.any():
            d = (tl[m, 3] - tl[m, 2]) / 1e6; e = (tl[m, 3] - t0) / 1e6
            print(f"  first 2.5 ms {names[ty]:8s} n={m.sum():5d} dur p50 {np.median(d):.3f} max {d.max():.3f} ms; ends p50 {np.median(e):.3f} max {e.max():.3f} ms")
