"""Bounds-checked build (libxdrop_checked.so, -DXDROP_CHECKED): every packed-pool word any kernel
reads must lie inside a pool registered for the call, else the kernel traps.  Runs in a child process
(a trap poisons the CUDA context) over ragged reads, seeds at both read ends, reverse-complement
pairs, every forced path and both packed kernels, and still checks the answers against the oracle.
"""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_CHECKED = os.path.join(ROOT, "paper_2309_07270_b200", "libxdrop_checked.so")


def child_env(lib, **extra):
    """The child's environment: the library under test plus the repo on PYTHONPATH, APPENDED to the
    inherited one (the driver's load hooks travel in the parent's environment)."""
    pp = os.environ.get("PYTHONPATH", "")
    return {**os.environ, "XDROP_LIB": lib, "PYTHONPATH": ROOT + (os.pathsep + pp if pp else ""), **extra}


@pytest.fixture(scope="module")
def checked_lib():
    """libxdrop_checked.so, built here if missing (every test of this module uses it)."""
    sys.path.insert(0, os.path.join(ROOT, "paper_2309_07270_b200"))
    try:
        import build as B
        B.build_checked(verbose=True)
    finally:
        sys.path.pop(0)
    return LIB_CHECKED

CHILD = textwrap.dedent("""
    import numpy as np
    import oracle
    import paper_2309_07270_b200 as xd
    from paper_2309_07270_b200 import _native
    from synth import workload as W
    assert _native.LIB_PATH.endswith("libxdrop_checked.so"), _native.LIB_PATH
    F = ("score", "a_begin", "a_end", "b_begin", "b_end")

    def run(w, X, **kw):
        with xd.Aligner(**kw) as al:
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
        ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, w.M, w.mu, w.g, X)
        for f in F:
            assert np.array_equal(res[f], ref[f]), (kw, X, f)
        assert np.array_equal(cells, rc), (kw, X, "cells")

    n = 0
    for flags in (0, 1, 2, 4, 8, 16):
        for X in (0, 15, 50):
            w = W.random_pairs_workload(seed=300 + flags + X, n_pairs=40 if flags == 2 else 120, len_lo=0,
                                        len_hi=600, k=11, X=X, rc_frac=0.3)
            run(w, X, flags=flags); n += 1
    w = W.random_pairs_workload(seed=77, n_pairs=8, len_lo=1500, len_hi=2500, k=11, X=300)
    for kernel in ("tiered", "shared"):
        run(w, 300, kernel=kernel); n += 1
    w = W.config("cfg1")
    run(w, w.X); n += 1
    # unrelated continuations at X = 500 (packed path) outgrow S = 1024: the packed S = 2048 level
    # (pk_wide_kernel) and the 32-bit S = 4096 level read the pool through the checker too
    w = W.random_pairs_workload(seed=661, n_pairs=12, len_lo=6000, len_hi=8000, k=11, X=500, related=0.0)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=500)
        assert al.stats()["cta_items"] > 0
    ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, w.M, w.mu, w.g, 500)
    assert all(np.array_equal(res[f], ref[f]) for f in F) and np.array_equal(cells, rc)
    n += 1
    # the compat mode: general-path kernels (8-lane group first, warp ring first), packed tiers (X = 500)
    import os
    wc = W.random_pairs_workload(seed=662, n_pairs=60, len_lo=0, len_hi=800, k=11, X=15, rc_frac=0.3)
    for first, X, w in (("1", 15, wc), ("2", 15, wc),
                        ("0", 500, W.random_pairs_workload(seed=663, n_pairs=4, len_lo=3000, len_hi=4000, k=11,
                                                           X=500, related=0.0))):
        os.environ["XDROP_COMPAT_FIRST"] = first
        os.environ["XDROP_COMPAT_GENERAL"] = "1" if first != "0" else "0"   # "0": the packed compat path
        with xd.Aligner(seqan_compat=True) as al:
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
            if X == 500:
                assert al.stats()["escalated"][2] > 0
        ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, w.M, w.mu, w.g, X,
                                     compat=True)
        assert all(np.array_equal(res[f], ref[f]) for f in F) and np.array_equal(cells, rc)
        n += 1
    print("checked ok", n)
""")


def test_checked_build_every_path(checked_lib):
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=child_env(checked_lib))
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "checked ok 25" in r.stdout


def test_checked_build_traps_out_of_bounds_reads(checked_lib):
    """The checker itself: with only the guard band registered, the first real read must trap and the
    call must fail with XDROP_ECUDA (-3), not return results."""
    child = textwrap.dedent("""
        import paper_2309_07270_b200 as xd
        from synth import workload as W
        w = W.config("tiny")
        try:
            with xd.Aligner() as al:
                al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
            print("no trap")
        except xd.XdropError as e:
            print("status", e.status)
    """)
    r = subprocess.run([sys.executable, "-c", child], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=child_env(checked_lib, XDROP_CHK_SHRINK="1"))
    assert "status -3" in r.stdout.split("\n"), (r.stdout[-2000:], r.stderr[-2000:])


CHILD_FULL = textwrap.dedent("""
    import numpy as np
    import oracle
    import paper_2309_07270_b200 as xd
    from synth import workload as W
    F = ("score", "a_begin", "a_end", "b_begin", "b_end")
    for name, scale, X in (("ecoli", 1.0, None), ("celegans", 0.01, None), ("xsweep", 0.05, 100)):
        w = W.config(name, scale=scale, X=X)
        with xd.Aligner() as al:
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        # E. coli (the benched batch): every pair; the others: 600 evenly spaced pairs
        n_chk = w.n_pairs if name == "ecoli" else min(w.n_pairs, 600)
        idx = np.linspace(0, w.n_pairs - 1, n_chk).astype(np.int64)
        ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs[idx], w.k, w.M, w.mu, w.g, w.X)
        for f in F:
            assert np.array_equal(res[f][idx], ref[f]), (name, f)
        assert np.array_equal(cells[idx], rc), (name, "cells")
        print(name, w.n_pairs, "ok", flush=True)
    print("full ok")
""")


def test_checked_build_config_workloads(checked_lib):
    """The bench's full E. coli-shaped batch (the launch configuration bench.py times; every pair
    bit-exact) and small C. elegans-shaped / X = 100 sweep batches (sampled pairs bit-exact) through
    the bounds-checked build: no trap."""
    r = subprocess.run([sys.executable, "-c", CHILD_FULL], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=child_env(checked_lib))
    assert r.returncode == 0 and "full ok" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
