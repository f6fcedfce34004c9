"""Scratch: per-anti-diagonal live-window span of X-drop extensions (numpy; not the oracle).

Prints, for spurious vs related extensions of a workload, the distribution of the window a tier
needs (span of live cells of anti-diagonals d-1 and d, in cells) weighted by anti-diagonals,
and each extension's lifetime maximum -- the quantity that decides escalation.
  python tools/band_profile.py [celegans|xsweep] [n_ext] [X]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import workload as W

NEG = -10 ** 9


def spans(a, b, M=1, mu=-1, g=-1, X=15):
    m, n = len(a), len(b)
    H1 = np.full(m + 2, NEG, np.int64); H2 = np.full(m + 2, NEG, np.int64)   # index i+1
    H1[1] = 0
    best = 0
    out = []
    live1 = (0, 0); live2 = None
    for d in range(1, m + n + 1):
        if live1 is None and live2 is None:
            break
        los = []; his = []
        if live1: los.append(live1[0]); his.append(live1[1] + 1)
        if live2: los.append(live2[0] + 1); his.append(live2[1] + 1)
        lo = max(0, d - n, min(los)); hi = min(m, d, max(his))
        H0 = np.full(m + 2, NEG, np.int64)
        if hi >= lo:
            i = np.arange(lo, hi + 1)
            j = d - i
            up = H1[i] + g                     # (i-1, j): index i-1+1 = i
            left = np.where(j >= 1, H1[i + 1] + g, NEG)
            ok = (i >= 1) & (j >= 1)
            ai = np.where(ok, a[np.maximum(i - 1, 0)], 0); bj = np.where(ok, b[np.maximum(j - 1, 0)], 0)
            diag = np.where(ok, H2[i] + np.where(ai == bj, M, mu), NEG)
            v = np.maximum(np.maximum(up, left), diag)
            v = np.where(v < NEG // 2, NEG, v)
            livem = (v >= best - X) & (v > NEG // 2)
            H0[i + 1] = np.where(livem, v, NEG)
            if livem.any():
                li = i[livem]
                newl = (int(li.min()), int(li.max()))
                vs = int(v[livem].max())
            else:
                newl = None; vs = None
        else:
            newl = None; vs = None
        if vs is not None and vs > best:
            best = vs
        live2, live1 = live1, newl
        # window needed for (d-1, d): diagonal span k = 2i - d of both live sets, in cells (diag/2)
        ks = []
        if live1: ks += [2 * live1[0] - d, 2 * live1[1] - d]
        if live2: ks += [2 * live2[0] - (d - 1), 2 * live2[1] - (d - 1)]
        if ks:
            out.append((max(ks) - min(ks)) // 2 + 1)
        H2, H1 = H1, H0
    return np.array(out)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "celegans"
    n_ext = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    X = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    w = W.config(name, scale=0.002) if name == "celegans" else W.config(name, scale=0.05)
    nr0 = w.recipe["n_reads"] - int(round(w.recipe["f_sp"] * w.n_pairs))
    sp = np.nonzero(w.pairs[:, 1] >= nr0)[0]
    rel = np.nonzero(w.pairs[:, 1] < nr0)[0]
    seq = np.frombuffer(w.seq, np.uint8) if isinstance(w.seq, (bytes, bytearray)) else np.asarray(w.seq)
    for label, idx in (("spurious", sp), ("related", rel)):
        allw = []; maxes = []
        for p in idx[:n_ext // 2]:
            a_id, b_id, pa, pb = (int(x) for x in w.pairs[p])
            A = seq[w.offsets[a_id]:w.offsets[a_id + 1]]; B = seq[w.offsets[b_id]:w.offsets[b_id + 1]]
            for a, b in ((A[pa + w.k:], B[pb + w.k:]), (A[:pa][::-1], B[:pb][::-1])):
                s = spans(a, b, X=X)
                if len(s):
                    allw.append(s); maxes.append(s.max())
        allw = np.concatenate(allw)
        qs = np.percentile(allw, [50, 90, 99, 100])
        print(f"{label}: anti-diagonals {len(allw)}; window need p50/p90/p99/max {qs}; "
              f"work fraction fitting 32/64/128/256: "
              + " ".join(f"{(allw <= c).mean():.3f}" for c in (30, 62, 126, 254))
              + f"; lifetime max per ext {sorted(maxes)}")


if __name__ == "__main__":
    main()
