"""CPU-only checks of the C-ABI library: it loads, exports every declared symbol, and its
host-side scheduler logic follows PAPER.md §III / Alg. 1 (SPEC.md test vectors)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def xd():
    from paper_2309_07270_b200 import build
    build.build()
    import paper_2309_07270_b200 as xd
    return xd


def test_exports_every_declared_symbol(xd):
    from paper_2309_07270_b200 import _native as N
    hdr = open(os.path.join(ROOT, "include", "xdrop.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(xdrop_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 12
    for name in sorted(declared):
        assert hasattr(N.lib, name), name
    assert declared <= set(N.EXPORTS) | declared
    assert set(N.EXPORTS) <= declared


def test_binding_constants_match_header(xd):
    """The binding's flag / policy values are the header's (the C ABI is the contract)."""
    from paper_2309_07270_b200 import _native as N
    hdr = open(os.path.join(ROOT, "include", "xdrop.h")).read()
    flags = {k: int(v) for k, v in re.findall(r"^#define XDROP_FLAG_(\w+)\s+(\d+)", hdr, re.M)}
    assert flags == {"FORCE_WIDE": N.FLAG_FORCE_WIDE, "FORCE_GENERAL": N.FLAG_FORCE_GENERAL,
                     "NO_SORT": N.FLAG_NO_SORT, "TIERED": N.FLAG_TIERED, "SHARED": N.FLAG_SHARED,
                     "SEQAN_COMPAT": N.FLAG_SEQAN_COMPAT}
    pol = {k.lower(): int(v) for k, v in re.findall(r"XDROP_POLICY_(\w+)\s*=\s*(\d+)", hdr)}
    assert all(N.POLICIES[k] == v for k, v in pol.items()) and len(pol) == 4


def test_strerror_and_no_device_fails_loudly(xd):
    from paper_2309_07270_b200 import _native as N
    assert N.lib.xdrop_strerror(-4) == b"base outside {A,C,G,T}"
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(xd.XdropError) as e:
            xd.Aligner()
        assert e.value.status == N.ENODEV


def test_ring_vectors_spec(xd):
    # SPEC.md:227-239 (Alg. 1 l.18-30 literal while-loops)
    assert xd.ring_left(2, 1, [3, 3, 3, 3]) == 1
    assert xd.ring_left(0, 1, [3, 3, 3, 3]) == 3
    assert xd.ring_left(2, 3, [3, 2, 3, 1]) == 0
    assert xd.ring_left(1, 5, [2, 5, 3]) is None
    assert xd.ring_right(2, 1, [3, 3, 3, 3]) == 3
    assert xd.ring_right(3, 1, [3, 3, 3, 3]) == 0
    assert xd.ring_right(0, 3, [3, 2, 3, 1]) == 2


def check_trace(trace, n_pairs, m, policy, n_ranks):
    assert trace["n_pairs"].sum() == n_pairs                     # exactly once
    for g in range(m):                                           # mutual exclusion per GPU
        ev = np.sort(trace[trace["gpu"] == g], order="t0_ms")
        assert np.all(ev["t0_ms"][1:] >= ev["t1_ms"][:-1] - 1e-9)
    if policy in ("one2one", "opt_one2one"):                     # pipeline affinity r mod m
        assert np.all(trace["gpu"] == trace["rank"] % m)
    if policy == "one2all":                                      # one rank at a time
        by_turn = {}
        for e in trace:
            key = (e["rank"], e["batch"], e["sub"])
            lo, hi = by_turn.get(key, (1e18, -1e18))
            by_turn[key] = (min(lo, e["t0_ms"]), max(hi, e["t1_ms"]))
        iv = sorted(by_turn.values())
        for a, b in zip(iv, iv[1:]):
            assert b[0] >= a[1] - 1e-9
    for r in range(n_ranks):                                     # per-rank order (batch, sub)
        ev = np.sort(trace[trace["rank"] == r], order="t0_ms")
        keys = list(zip(ev["batch"], ev["sub"]))
        assert keys == sorted(keys)


@pytest.mark.parametrize("policy", ["one2all", "one2one", "opt_one2one", "cells"])
def test_policies_randomized_deadlock_free(xd, policy):
    rng = np.random.default_rng(3)
    for _ in range(25):
        m = int(rng.integers(1, 5))
        n_ranks = int(rng.integers(1, 9))
        c = int(rng.integers(1, 4))
        bs = int(rng.integers(1, 9))
        n = int(rng.integers(0, 60))
        w = rng.integers(1, 100, size=n)
        trace, st, gpu = xd.sched_simulate(m, policy, n_ranks, w, batch_size=bs, subbatches=c, ns_per_unit=200)
        check_trace(trace, n, m, policy, n_ranks)
        assert np.all(gpu >= 0) or n == 0


def test_skewed_batch_counts_no_deadlock(xd):
    """Counts like [2,2,1] deadlock Alg. 1 read literally (Q21); ours must finish."""
    w = np.ones(5, dtype=np.int64)
    trace, st, _ = xd.sched_simulate(1, "one2all", 3, w, batch_size=1, subbatches=1)
    assert trace["n_pairs"].sum() == 5
    assert [int(r) for r in np.sort(trace, order="t0_ms")["rank"]] == [0, 1, 2, 0, 1]


def test_message_proportionality(xd):
    """§III-D: one2one sends per sub-batch, opt_one2one per batch."""
    for c in (1, 2, 5):
        for n_ranks in (2, 4):
            n = n_ranks * 3 * 10                       # 3 batches of 10 per rank
            w = np.ones(n, dtype=np.int64)
            _, s1, _ = xd.sched_simulate(1, "one2one", n_ranks, w, batch_size=10, subbatches=c)
            _, s2, _ = xd.sched_simulate(1, "opt_one2one", n_ranks, w, batch_size=10, subbatches=c)
            turns1, turns2 = n_ranks * 3 * c, n_ranks * 3
            assert s1["handoffs"] == turns1 - 1 and s2["handoffs"] == turns2 - 1
            assert s1["exchange_msgs"] == s2["exchange_msgs"] == n_ranks * (n_ranks - 1)


def test_one2one_concurrency_and_cells_balance(xd):
    w = np.ones(400, dtype=np.int64)
    _, st, _ = xd.sched_simulate(4, "one2one", 8, w, batch_size=25, subbatches=2, ns_per_unit=20000)
    assert st["max_concurrent"] >= 2
    rng = np.random.default_rng(1)
    w = rng.integers(1, 1000, size=1000)
    _, _, gpu = xd.sched_simulate(4, "cells", 1, w)
    loads = np.bincount(gpu, weights=w, minlength=4)
    assert loads.max() - loads.min() <= w.max()                   # LPT bound


def _sass_opcode_counts(cubin):
    """{function: {opcode: count}} of a cubin (cuobjdump -sass)."""
    import subprocess
    txt = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True, check=True).stdout
    out, fn = {}, None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            out[fn] = {}
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
        if m and fn:
            out[fn][m.group(1)] = out[fn].get(m.group(1), 0) + 1
    return out


def test_peak_probes_sass(tmp_path):
    """The roofline denominators (csrc/xdrop_peaks.cu): each probe's loop is the ONE named SASS
    instruction (>= 95% of the kernel's instructions; 80% for the two-pipe mix, whose loop ptxas does not unroll further), so its measured rate is that pipe's rate."""
    import subprocess
    cubin = str(tmp_path / "peaks.cubin")
    subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-o",
                    cubin, os.path.join(ROOT, "paper_2309_07270_b200", "csrc", "xdrop_peaks.cu")], check=True)
    counts = _sass_opcode_counts(cubin)
    want = {"0": {"VIMNMX3.S16x2"}, "1": {"VIMNMX3"}, "2": {"LOP3.LUT"}, "3": {"IADD3"}, "4": {"IMAD"},
            "5": {"VIMNMX3.S16x2", "IMAD"}}
    seen = set()
    for fn, c in counts.items():
        m = re.search(r"peak_kernelILi(\d)E", fn)
        if not m:
            continue
        seen.add(m.group(1))
        total = sum(c.values())
        named = sum(v for k, v in c.items() if k in want[m.group(1)])
        # (the mix loop is not unrolled further by ptxas: ~55 prologue/epilogue instructions around the 257-instruction loop)
        assert named >= (0.8 if m.group(1) == "5" else 0.95) * total, (m.group(1), c)
        if m.group(1) == "5":
            assert abs(c["IMAD"] - c["VIMNMX3.S16x2"]) <= 0.05 * named, c
    assert seen == set(want), seen


def test_new_entry_points_argument_errors(xd):
    """Argument checks of the round-2 entry points that need no GPU: bad sizes / parameters return
    XDROP_EINVAL before any CUDA call (include/xdrop.h)."""
    import ctypes
    from paper_2309_07270_b200 import _native as N
    out = (ctypes.c_double * 4)()
    assert N.lib.xdrop_alu_peaks(0, out, 4) == N.EINVAL                      # n_out < 12
    assert N.lib.xdrop_alu_peaks(0, None, 12) == N.EINVAL
    err = ctypes.c_int64(7)
    # adaptive filter: phi must be > 0, c >= 0; n < 0 invalid; n == 0 is a no-op
    assert N.lib.xdrop_adaptive_filter_device(None, 0, None, 0, None, None, 0, 0.0, 1.0, None,
                                              ctypes.byref(err), None) == N.EINVAL
    assert N.lib.xdrop_adaptive_filter_device(None, 0, None, 0, None, None, -1, 0.5, 1.0, None, None, None) == N.EINVAL
    assert N.lib.xdrop_adaptive_filter_device(None, 0, None, 0, None, None, 0, 0.5, 1.0, None,
                                              ctypes.byref(err), None) == N.OK
    assert err.value == -1
    # k-mer band: 1 <= k <= 31; n == 0 is a no-op; a NULL pointer with n > 0 is invalid
    assert N.lib.xdrop_seed_kmer_freq_device(None, None, 0, 0, None, 0, 32, 0, 1, None, None, None, None) == N.EINVAL
    assert N.lib.xdrop_seed_kmer_freq_device(None, None, 0, 0, None, 0, 17, 0, 1, None, None, None, None) == N.OK
    assert N.lib.xdrop_seed_kmer_freq_device(None, None, 0, 0, None, 5, 17, 0, 1, None, None, None, None) == N.EINVAL
    # ring order helpers: a consistent next / prev walk over a skewed ring (reading Q21)
    counts = (ctypes.c_int * 3)(2, 2, 1)
    nb, nit = ctypes.c_int(0), ctypes.c_int(0)
    assert N.lib.xdrop_ring_turn_next(2, 1, 1, counts, 3, 1, ctypes.byref(nb), ctypes.byref(nit)) == 0
    assert (nb.value, nit.value) == (2, 1)                                 # batch 2 of member 0
    assert N.lib.xdrop_ring_turn_prev(0, 2, 1, counts, 3, 1) == 2
    assert N.lib.xdrop_ring_turn_next(1, 2, 1, counts, 3, 1, None, None) == -1
