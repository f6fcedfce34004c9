"""GPU parity of the SeqAn/LOGAN-style compat mode (XDROP_FLAG_SEQAN_COMPAT; SURVEY.md §8(f) f3,
DESIGN.md readings Q28-Q30) against the CPU oracle's compat mode, bit-exact on every field and the
cell count: the hand-traced fixtures embedded as right extensions, ragged random pairs (seeds at
read ends, RC pairs, several X and scoring schemes), an E. coli-shaped batch and the X-sweep shape,
and the device / pooled entry points."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("score", "a_begin", "a_end", "b_begin", "b_end")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def xd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2309_07270_b200 as xd
    return xd


def oracle_compat(seq, off, pairs, k, X, M=1, mu=-1, g=-1):
    import oracle
    return oracle.align_batch(seq, off, seq, off, pairs, k, M=M, mu=mu, g=g, X=X, compat=True)


def assert_same(res, cells, ref, rcells, what):
    for f in FIELDS:
        bad = np.nonzero(res[f] != ref[f])[0]
        assert bad.size == 0, f"{what}: {f} differs at {bad[:10]} gpu={res[bad[:5]]} ref={ref[bad[:5]]}"
    bad = np.nonzero(cells != rcells)[0]
    assert bad.size == 0, f"{what}: cells differ at {bad[:10]}: {cells[bad[:5]]} vs {rcells[bad[:5]]}"


def test_compat_hand_fixtures(xd):
    """Each row of tests/golden/extend_compat_hand.txt as the right extension of a pair whose seed
    starts both reads (the left extension is empty): score = seed + H, a_end = k + i, b_end = k + j."""
    import oracle
    rows = []
    with open(os.path.join(GOLDEN, "extend_compat_hand.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                lhs, rhs = line.split("|")
                a, b, M, mu, g, X = lhs.split()
                rows.append(("" if a == "-" else a, "" if b == "-" else b, int(M), int(mu), int(g), int(X),
                             [int(t) for t in rhs.split()]))
    seed = "GATTACAGATTACAGAT"
    k = len(seed)
    for a, b, M, mu, g, X, (H, i, j, c) in rows:
        reads = [(seed + a).encode(), (seed + b).encode()]
        seq = np.frombuffer(b"".join(reads), dtype=np.uint8)
        off = np.array([0, len(reads[0]), len(reads[0]) + len(reads[1])], dtype=np.int64)
        pairs = np.array([[0, 1, 0, 0]], dtype=np.int32)
        with xd.Aligner(seqan_compat=True) as al:
            res, cells = al.align(seq, off, pairs, k=k, X=X, M=M, mu=mu, g=g)
        want = (k * M + H, 0, k + i, 0, k + j)
        assert tuple(int(res[f][0]) for f in FIELDS) == want, (a, b, X)
        assert int(cells[0]) == 1 + c, (a, b, X)      # + the empty left extension's origin
        ref, rc = oracle.align_batch(seq, off, seq, off, pairs, k, M=M, mu=mu, g=g, X=X, compat=True)
        assert_same(res, cells, ref, rc, f"fixture {a}/{b}")


@pytest.mark.parametrize("path", ["packed", "group", "ring"])
@pytest.mark.parametrize("X", [0, 1, 5, 15, 100])
def test_compat_random_ragged(xd, X, path, monkeypatch):
    """packed: the default compat path (packed tiers with the Q28 edge kill and the Q29 last maximum,
    S > 1024 restarting in the general path); group / ring: XDROP_COMPAT_GENERAL=1, the general path
    only, with the 8-lane group kernel (256-cell rings) or the warp-ring kernel first."""
    from synth import workload as W
    first = {"packed": "0", "group": "1", "ring": "2"}[path]
    if path != "packed":
        monkeypatch.setenv("XDROP_COMPAT_GENERAL", "1")
    monkeypatch.setenv("XDROP_COMPAT_FIRST", first)
    w = W.random_pairs_workload(seed=900 + X, n_pairs=300, len_lo=0, len_hi=1500, k=11, X=X, rc_frac=0.3)
    with xd.Aligner(seqan_compat=True) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
        st = al.stats()
    if first == "1" and X == 100:
        assert st["escalated"][1] > 0          # some hulls outgrew the group's ring
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, X)
    assert_same(res, cells, ref, rcells, f"compat random X={X} path={path}")


@pytest.mark.parametrize("general", ["0", "1"])
@pytest.mark.parametrize("M,mu,g", [(2, -3, -2), (1, -2, -1), (5, -4, -3)])
def test_compat_scoring(xd, M, mu, g, general, monkeypatch):
    from synth import workload as W
    monkeypatch.setenv("XDROP_COMPAT_GENERAL", general)
    monkeypatch.setenv("XDROP_COMPAT_FIRST", "1")
    w = W.random_pairs_workload(seed=950 + M, n_pairs=200, len_lo=0, len_hi=800, k=9, X=12, rc_frac=0.2)
    with xd.Aligner(seqan_compat=True) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=12, M=M, mu=mu, g=g)
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, 12, M, mu, g)
    assert_same(res, cells, ref, rcells, f"compat scoring {(M, mu, g)}")


def test_compat_differs_from_default(xd):
    """The flag changes the answer where Q28-Q30 say it must: on spurious continuations the longest
    extension lies past the best cell, so compat scores are lower and ends later."""
    from synth import workload as W
    w = W.config("ecoli", scale=0.02)
    with xd.Aligner() as al:
        r0, c0 = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    with xd.Aligner(seqan_compat=True) as al:
        r1, c1 = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    # H at the longest extension is at most the extension's best (the edge rule can in principle
    # change which cells live, so "at most the default mode's" is only nearly always true)
    assert (r1["score"] != r0["score"]).any()
    assert (r1["score"] <= r0["score"]).mean() > 0.99
    assert (r1["a_end"] >= r0["a_end"]).mean() > 0.5
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, w.X)
    assert_same(r1, c1, ref, rcells, "compat ecoli x0.02")


def test_compat_ecoli_and_xsweep_shapes(xd):
    """5,000 E. coli-shaped pairs and 500 X-sweep-shaped pairs (20 kb, 20 % spurious) at X = 50 and
    X = 100; at X = 100 some hulls outgrow the warp's shared-memory ring (1,024 cells) and are redone
    by the 8-warp ring kernel (stats()["escalated"][2])."""
    from synth import workload as W
    for name, scale, X in [("ecoli", 0.05, 15), ("xsweep", 0.05, 50), ("xsweep", 0.05, 100)]:
        w = W.config(name, scale=scale).with_X(X)
        with xd.Aligner(seqan_compat=True) as al:
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
            st = al.stats()
        ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, X)
        assert_same(res, cells, ref, rcells, f"compat {name} X={X}")
        print(f"compat {name} x{scale} X={X}: {cells.sum() / st['kernel_ms'] / 1e6:.1f} GCUPS "
              f"({st['kernel_ms']:.1f} ms kernel, ring overflows {st['escalated'][2:]})")
        if X == 100:
            assert st["escalated"][2] > 0


def test_compat_unbounded_hulls(xd):
    """Unrelated 12 kb reads seeded at their first base, X = 12,000: the right extension's hull grows
    to the full anti-diagonal (> 8,192 cells), past both shared-memory rings, so it ends in the
    global-memory kernel; still bit-exact."""
    rng = np.random.default_rng(990)
    k, L = 11, 12_000
    reads = []
    for _ in range(2):
        a = rng.integers(0, 4, size=L, dtype=np.uint8)
        b = rng.integers(0, 4, size=L - 300, dtype=np.uint8)
        b[:k] = a[:k]
        reads += [a, b]
    seq = np.frombuffer(b"".join(np.frombuffer(b"ACGT", dtype=np.uint8)[r].tobytes() for r in reads), dtype=np.uint8)
    off = np.concatenate([[0], np.cumsum([r.shape[0] for r in reads])]).astype(np.int64)
    pairs = np.array([[0, 1, 0, 0], [2, 3, 0, 0]], dtype=np.int32)
    with xd.Aligner(seqan_compat=True) as al:
        res, cells = al.align(seq, off, pairs, k=k, X=L)
        st = al.stats()
    assert st["escalated"][3] > 0
    ref, rcells = oracle_compat(seq, off, pairs, k, L)
    assert_same(res, cells, ref, rcells, "compat unbounded")


def test_compat_device_and_pooled(xd):
    import torch
    from synth import workload as W
    w = W.random_pairs_workload(seed=977, n_pairs=250, len_lo=20, len_hi=1200, k=13, X=20, rc_frac=0.3)
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, 20)
    with xd.Aligner(seqan_compat=True) as al:
        dev = torch.device("cuda:0")
        seq = torch.from_numpy(w.seq).to(dev)
        off = torch.from_numpy(w.offsets).to(dev)
        pairs = torch.from_numpy(w.pairs).to(dev)
        out = torch.empty((w.n_pairs, 5), dtype=torch.int32, device=dev)
        cells = torch.empty(w.n_pairs, dtype=torch.int64, device=dev)
        al.align_device(seq, off, pairs, out, cells, k=w.k, X=20)
        o = out.cpu().numpy()
        res = np.zeros(w.n_pairs, dtype=ref.dtype)
        for t, f in enumerate(FIELDS):
            res[f] = o[:, t]
        assert_same(res, cells.cpu().numpy(), ref, rcells, "compat device API")
        pid = al.register_pool(w.seq, w.offsets)
        res2, cells2 = al.align_pooled(pid, w.pairs, k=w.k, X=20)
        assert_same(res2, cells2, ref, rcells, "compat pooled API")


def _device_run(xd, w, **kw):
    import torch
    dev = torch.device("cuda:0")
    seq = torch.from_numpy(w.seq).to(dev)
    off = torch.from_numpy(w.offsets).to(dev)
    pairs = torch.from_numpy(w.pairs).to(dev)
    out = torch.full((w.n_pairs, 5), -7, dtype=torch.int32, device=dev)
    cells = torch.full((w.n_pairs,), -7, dtype=torch.int64, device=dev)
    with xd.Aligner(devices=[0], seqan_compat=True) as al:
        for _ in range(2):                                   # a warm context, as the bench runs it
            al.align_device(seq, off, pairs, out, cells, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)
    torch.cuda.synchronize(dev)
    o = out.cpu().numpy()
    res = np.zeros(w.n_pairs, dtype=xd.RESULT_DTYPE)
    for i, f in enumerate(FIELDS):
        res[f] = o[:, i]
    return res, cells.cpu().numpy()


@pytest.mark.parametrize("name,X", [("ecoli", 15), ("xsweep", 15), ("xsweep", 50), ("xsweep", 100)])
def test_compat_every_pair_configs_2_4(xd, name, X):
    """Compat mode on EVERY pair of BASELINE configs 2 and 4 (the packed CP tiers, S = 2048 and the
    general-path restarts included), bit-exact against the oracle's compat mode."""
    from synth import workload as W
    w = W.config(name).with_X(X)
    res, cells = _device_run(xd, w)
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, X)
    assert_same(res, cells, ref, rcells, f"compat every pair {name} X={X}")


def test_compat_multiseed(xd):
    """xdrop_align_multiseed in the compat mode: every seed row aligned with Q28-Q30 and the best
    seed chosen on those scores (Q26 on the compat scores), against the oracle's."""
    import oracle
    from synth import workload as W
    w = W.make_pool_workload("ms-compat", 92, 200_000, 150, W._normal_len(2000, 300, 800, 4000), 8.0, 300,
                             k=15, X=15, rc_frac=0.3, seeds_per_pair=3, f_sp=0.1)
    ref, rcells = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, X=w.X, compat=True)
    rbest = oracle.best_seed(w.pairs, ref["score"])
    with xd.Aligner(seqan_compat=True) as al:
        res, best, cells = al.align_multiseed(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    assert_same(res, cells, ref, rcells, "compat multiseed")
    assert np.array_equal(best, rbest)


@pytest.mark.parametrize("flags", [1, 2, 4, 8, 16])
def test_compat_with_test_flags(xd, flags):
    """Compat mode combined with every other XDROP_FLAG_* (FORCE_WIDE is ignored: the 32-bit warp level
    has no compat instance; FORCE_GENERAL runs the unbounded kernel; NO_SORT, TIERED, SHARED as named)."""
    from synth import workload as W
    w = W.random_pairs_workload(seed=1300 + flags, n_pairs=120, len_lo=0, len_hi=1200, k=11, X=20, rc_frac=0.3)
    with xd.Aligner(seqan_compat=True, flags=flags) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=20)
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, 20)
    assert_same(res, cells, ref, rcells, f"compat flags={flags}")


@pytest.mark.parametrize("policy,n_ranks", [("cells", 1), ("one2all", 4), ("one2one", 4), ("opt_one2one", 4)])
def test_compat_policies_logical_devices(xd, policy, n_ranks):
    """The compat mode under every scheduler policy on three logical devices (streams of GPU 0):
    results identical to the oracle's compat mode."""
    from synth import workload as W
    w = W.config("cfg1")
    with xd.Aligner(devices=[0, 0, 0], policy=policy, n_ranks=n_ranks, batch_size=37, seqan_compat=True) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    ref, rcells = oracle_compat(w.seq, w.offsets, w.pairs, w.k, w.X)
    assert_same(res, cells, ref, rcells, f"compat {policy}")
