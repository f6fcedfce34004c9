"""Config 5 (C. elegans-shaped, 5M pairs) at full scale on one GPU, with a stratified oracle sample
(every 100th pair in cost order plus the 1,000 longest).

  python tools/celegans_full.py [--scale 1.0] [--out profiles/celegans_full_r1.md]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd  # noqa: E402
from synth import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t0 = time.time()
    w = W.config("celegans", scale=a.scale)
    gen_s = time.time() - t0
    p = w.pairs.reshape(-1, 4)
    lines = [f"# Config 5 (C. elegans-shaped) at scale {a.scale} on one B200", "",
             f"generated in {gen_s:.0f} s: {p.shape[0]} pairs, {len(w.offsets) - 1} reads, "
             f"{w.seq.shape[0] / 1e9:.2f} Gb pool", ""]
    with xd.Aligner() as al:
        ts = []
        for _ in range(3):
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            st = al.stats()
            ts.append((st["total_ms"], st["level_ms"], st["band_kernel"]))
    best = min(ts, key=lambda x: x[0])
    tot = float(cells.sum())
    lines += ["| pairs | cells | device ms | GCUPS | alignments/s | tier ms (T0-2 / S1024 / - / unbounded) | checkpoints | band kernel |",
              "|---|---|---|---|---|---|---|---|",
              f"| {p.shape[0]} | {tot:.3e} | {best[0]:.1f} | {tot / best[0] / 1e6:.1f} | {p.shape[0] / best[0] * 1e3:.3e} | "
              f"{'/'.join('%.1f' % x for x in best[1])} | {st['escalated']} | {best[2]} |", "",
              "calls (device ms, kernel): " + ", ".join(f"{t[0]:.1f} {t[2]}" for t in ts), ""]
    # stratified oracle sample: every 100th pair in cost order + the 1,000 longest
    import oracle
    lens = np.diff(w.offsets)
    la, lb = lens[p[:, 0]], lens[p[:, 1] & 0x7fffffff]
    cost = np.minimum(p[:, 2], p[:, 3]) + np.minimum(la - p[:, 2] - w.k, lb - p[:, 3] - w.k)
    order = np.argsort(-cost, kind="stable")
    idx = np.unique(np.concatenate([order[::100], order[:1000]]))
    t1 = time.time()
    ref, rcells = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, p[idx], w.k, X=w.X)
    ok = bool(np.array_equal(res[idx], ref) and np.array_equal(cells[idx], rcells))
    lines += [f"oracle sample: {idx.shape[0]} pairs (every 100th in cost order + the 1,000 longest), "
              f"{rcells.sum():.3e} cells in {time.time() - t1:.0f} s on {os.cpu_count()} threads: "
              f"**{'bit-exact' if ok else 'MISMATCH'}**"]
    text = "\n".join(lines) + "\n"
    print(text)
    if a.out:
        open(a.out, "w").write(text)
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
