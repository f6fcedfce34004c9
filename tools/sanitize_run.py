"""Small workloads through every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck). Each batch is also checked bit-exact against the CPU oracle, so a run that the sanitizer
lets through still has to produce the right answers.

usage (GPU box): compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py [--quick]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: checks the answers)
import paper_2309_07270_b200 as xd  # noqa: E402
from synth import workload as W  # noqa: E402

FIELDS = ("score", "a_begin", "a_end", "b_begin", "b_end")


def check(w, res, cells, X, what):
    ref, rcells = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, w.M, w.mu, w.g, X)
    for f in FIELDS:
        assert np.array_equal(res[f], ref[f]), f"{what}: {f} differs"
    assert np.array_equal(cells, rcells), f"{what}: cells differ"


def main():
    quick = "--quick" in sys.argv
    cases = [(0, 15), (1, 15), (2, 5), (4, 15), (8, 50), (16, 50)]
    if quick:
        cases = [(0, 15), (16, 50), (2, 5)]
    for flags, X in cases:
        w = W.random_pairs_workload(seed=7 + flags, n_pairs=24 if flags == 2 else 48, len_lo=0, len_hi=400,
                                    k=11, X=X)
        with xd.Aligner(flags=flags) as al:
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
        check(w, res, cells, X, f"flags={flags} X={X}")
        print(f"flags={flags} X={X}: {w.n_pairs} pairs ok", flush=True)
    # wide bands that escalate past the warp tiers (unrelated continuations, large X)
    w = W.random_pairs_workload(seed=99, n_pairs=6, len_lo=1500, len_hi=2500, k=11, X=300)
    for kernel in ("tiered", "shared"):
        with xd.Aligner(kernel=kernel) as al:
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=300)
        check(w, res, cells, 300, f"wide {kernel}")
        print(f"wide X=300 {kernel}: ok", flush=True)
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
