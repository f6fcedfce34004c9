"""Throughput of the BASELINE.json configs on the GPUs available (no oracle here; parity of
the same configs lives in tests/test_gpu_configs.py and tests/test_gpu_parity.py).

  python tools/configs_bench.py [--celegans-scale 0.1] [--out profiles/configs_r1.md]

* config 1  (cfg1): 200 pairs, 1-2 kb
* config 2  (ecoli): 100k pairs, ~10 kb  (the bench.py workload)
* config 3  policies: the config-2 batch through one2all / one2one / opt_one2one with the paper's
            16 logical ranks and batch 10,000 on m logical devices
            (streams of the available GPU(s)) -- alignment span, handoffs, busy per device
* config 4  (xsweep): 10k pairs of 20 kb, f_sp 0.2, X in {15, 50, 100}; escalation per level and the
            count of pairs whose score is not monotone in X (Q25)
* config 5  (celegans): lognormal 2-40 kb, f_sp 0.1, at --celegans-scale of the 5M-pair batch
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_07270_b200 as xd  # noqa: E402
from synth import workload as W  # noqa: E402


def run(al, w, X=None, reps=3):
    X = w.X if X is None else X
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        r, c = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X, M=w.M, mu=w.mu, g=w.g)
        wall = time.perf_counter() - t
        st = al.stats()
        if best is None or st["total_ms"] < best[2]["total_ms"]:
            best = (r, c, st, wall)
    return best


def fmt_row(name, w, X, r, c, st, wall):
    ms = st["total_ms"]
    return (f"| {name} | {w.n_pairs} | {X} | {c.sum():.3e} | {ms:.2f} | {c.sum() / ms / 1e6:.1f} | "
            f"{w.n_pairs / ms * 1e3:.3e} | {'/'.join('%.1f' % x for x in st['level_ms'])} | {st['escalated']} | {st['long_items']} | "
            f"{wall * 1e3:.1f} |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--celegans-scale", type=float, default=0.05)
    ap.add_argument("--logical-devices", type=int, default=4)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="comma list of: cfg1,ecoli,xsweep,celegans,policies")
    args = ap.parse_args()
    lines = ["| config | pairs | X | cells | device ms (pipeline) | GCUPS | alignments/s | tier ms (T0-2 / S1024 / - / unbounded) | "
             "checkpoints (T0>T1, T1>T2, T2>S1024, unbounded restarts) | long-mode ext. | host-API wall ms (incl. H2D/D2H) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    only = set(args.only.split(",")) if args.only else {"cfg1", "ecoli", "xsweep", "celegans", "policies"}
    al = xd.Aligner()
    nonmono, w5, gen_s, wx = None, None, 0.0, None
    for name in [n for n in ["cfg1", "ecoli"] if n in only]:
        w = W.config(name)
        lines.append(fmt_row(name, w, w.X, *run(al, w)))
        print(lines[-1], flush=True)
    # config 4: X sweep
    if "xsweep" in only:
        wx = W.config("xsweep")
        scores = {}
        for X in (15, 50, 100):
            r, c, st, wall = run(al, wx, X=X, reps=2)
            scores[X] = r["score"].copy()
            lines.append(fmt_row("xsweep", wx, X, r, c, st, wall))
            print(lines[-1], flush=True)
        nonmono = int(np.sum((scores[50] < scores[15]) | (scores[100] < scores[50])))
    # config 5
    if "celegans" in only:
        t = time.perf_counter()
        w5 = W.config("celegans", scale=args.celegans_scale)
        gen_s = time.perf_counter() - t
        lines.append(fmt_row(f"celegans x{args.celegans_scale}", w5, w5.X, *run(al, w5, reps=2)))
        print(lines[-1], flush=True)
    al.close()
    if "policies" not in only:
        print("\n".join(lines))
        return
    # config 3: the paper's policies on logical devices
    w = W.config("ecoli")
    m = args.logical_devices
    pol = ["| policy | ranks | devices | c | span ms | handoffs | exchange msgs | max concurrent turns | GCUPS (span) |",
           "|---|---|---|---|---|---|---|---|---|"]
    ref = None
    for policy, c in [("cells", 1), ("one2all", 1), ("one2one", 1), ("opt_one2one", 1), ("one2one", 4),
                      ("opt_one2one", 4)]:
        with xd.Aligner(devices=[0] * m, policy=policy, n_ranks=16, batch_size=10000, subbatches=c) as a2:
            r, cc = a2.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            r, cc = a2.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            ss = a2.sched_stats()
        if ref is None:
            ref = (r, cc)
        assert np.array_equal(r, ref[0]) and np.array_equal(cc, ref[1]), "policy changed the results"
        pol.append(f"| {policy} | {16 if policy != 'cells' else 1} | {m} | {c} | {ss['span_ms']:.1f} | "
                   f"{ss['handoffs']} | {ss['exchange_msgs']} | {ss['max_concurrent']} | "
                   f"{cc.sum() / ss['span_ms'] / 1e6:.1f} |")
        print(pol[-1], flush=True)
    import torch
    gpu = torch.cuda.get_device_name(0)
    text = "\n".join([f"# Configs on {gpu} (1 physical GPU)", "", "## Throughput", ""] + lines + [
        "", f"X-sweep pairs whose score is NOT monotone in X (15 -> 50 -> 100): {nonmono} of {wx.n_pairs if wx else 0}",
        f"(DESIGN.md Q25: monotonicity is not a property of X-drop).", "",
        f"config 5 generated at scale {args.celegans_scale} in {gen_s:.1f} s "
        f"({w5.n_pairs if w5 else 0} pairs, {len(w5.offsets) - 1 if w5 else 0} reads).", "",
        f"## Config 3 analog: the paper's policies, 16 logical ranks over {m} logical devices", "",
        "Logical devices are streams of one B200, so spans show policy overheads and serialisation, not",
        "multi-GPU scaling. Results are identical for every policy (asserted).", ""] + pol) + "\n"
    print(text)
    if args.out:
        open(args.out, "w").write(text)


if __name__ == "__main__":
    main()
