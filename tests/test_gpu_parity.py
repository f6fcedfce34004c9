"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Fields compared element by element: score, a_begin, a_end, b_begin, b_end and
the DP cell count (integer work: the bar is bit-exactness).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("score", "a_begin", "a_end", "b_begin", "b_end")


@pytest.fixture(scope="module")
def xd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2309_07270_b200 as xd
    return xd


def oracle_of(w, pairs=None, X=None, M=None, mu=None, g=None):
    import oracle
    return oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs if pairs is None else pairs, w.k,
                              M=w.M if M is None else M, mu=w.mu if mu is None else mu,
                              g=w.g if g is None else g, X=w.X if X is None else X)


def assert_same(res, cells, ref, rcells, what=""):
    for f in FIELDS:
        bad = np.nonzero(res[f] != ref[f])[0]
        assert bad.size == 0, f"{what}: field {f} differs at pairs {bad[:10]} gpu={res[bad[:5]]} ref={ref[bad[:5]]}"
    bad = np.nonzero(cells != rcells)[0]
    assert bad.size == 0, f"{what}: cells differ at {bad[:10]}: {cells[bad[:5]]} vs {rcells[bad[:5]]}"


def test_cfg1_full(xd):
    from synth import workload as W
    w = W.config("cfg1")
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, "cfg1")


@pytest.mark.parametrize("flags", [0, 1, 2, 4, 8, 16])
@pytest.mark.parametrize("X", [0, 1, 5, 15, 50])
def test_random_edge_cases_all_paths(xd, flags, X):
    from synth import workload as W
    w = W.random_pairs_workload(seed=100 + X, n_pairs=150 if flags != 2 else 40, len_lo=0, len_hi=700,
                                k=11, X=X)
    with xd.Aligner(flags=flags) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
    ref, rcells = oracle_of(w, X=X)
    assert_same(res, cells, ref, rcells, f"random X={X} flags={flags}")


@pytest.mark.parametrize("M,mu,g", [(2, -3, -2), (5, -4, -3), (2, -1, -1), (1, -2, -1)])
def test_scoring_schemes(xd, M, mu, g):
    from synth import workload as W
    w = W.random_pairs_workload(seed=7 * M - mu, n_pairs=120, len_lo=20, len_hi=900, k=17, X=20,
                                M=M, mu=mu, g=g)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=17, X=20, M=M, mu=mu, g=g)
    ref, rcells = oracle_of(w, M=M, mu=mu, g=g)
    assert_same(res, cells, ref, rcells, f"scoring {M},{mu},{g}")


def test_unrelated_wide_bands_escalate(xd):
    """Unrelated continuations widen the band past the lane window (level 1/2 paths)."""
    from synth import workload as W
    w = W.random_pairs_workload(seed=5, n_pairs=60, len_lo=800, len_hi=2500, k=17, X=60, related=0.0)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=17, X=60)
        st = al.stats()
    ref, rcells = oracle_of(w, X=60)
    assert_same(res, cells, ref, rcells, "wide")
    assert st["escalated"][0] > 0


@pytest.mark.parametrize("s1024", ["0", "1"])
def test_cta_path_wide_band(xd, s1024, monkeypatch):
    """X large enough that nothing is pruned, hull 1000-3000 cells: checkpoints travel
    lane -> lane pair -> warp (256) -> warp (1024; or a 4-warp CTA with XDROP_S1024=1) -> CTA (4096)
    and resume exactly."""
    from synth import workload as W
    monkeypatch.setenv("XDROP_S1024", s1024)
    w = W.random_pairs_workload(seed=9, n_pairs=8, len_lo=1200, len_hi=3000, k=5, X=100000, related=0.0)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=5, X=100000)
        st = al.stats()
    ref, rcells = oracle_of(w, X=100000)
    assert_same(res, cells, ref, rcells, "cta")
    assert st["escalated"][2] > 0 and st["escalated"][3] == 0


def test_general_path_huge_band(xd):
    """Hull wider than the CTA window (4096 cells): the unbounded kernel restarts it."""
    from synth import workload as W
    w = W.random_pairs_workload(seed=19, n_pairs=3, len_lo=4500, len_hi=5000, k=5, X=100000, related=0.0)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=5, X=100000)
        st = al.stats()
    ref, rcells = oracle_of(w, X=100000)
    assert_same(res, cells, ref, rcells, "general")
    assert st["escalated"][3] > 0


def test_ecoli_shaped_sample_full_launch(xd):
    """Full E. coli-shaped batch in the bench's launch configuration; a sample is checked
    against the oracle (every 50th pair + the 200 longest), all checked for sanity."""
    from synth import workload as W
    w = W.config("ecoli")
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    lens = np.diff(w.offsets)
    est = np.minimum(w.pairs[:, 2], w.pairs[:, 3]) + np.minimum(lens[w.pairs[:, 0]] - w.pairs[:, 2],
                                                                 lens[w.pairs[:, 1]] - w.pairs[:, 3])
    idx = np.unique(np.concatenate([np.arange(0, w.n_pairs, 50), np.argsort(-est)[:200]]))
    ref, rcells = oracle_of(w, pairs=w.pairs[idx])
    assert_same(res[idx], cells[idx], ref, rcells, "ecoli sample")
    # properties at any size: seed inside the reported interval, score <= min span
    assert np.all(res["a_begin"] <= w.pairs[:, 2]) and np.all(res["a_end"] >= w.pairs[:, 2] + w.k)
    assert np.all(res["score"] <= np.minimum(res["a_end"] - res["a_begin"], res["b_end"] - res["b_begin"]))


@pytest.mark.parametrize("policy,n_ranks,c", [("cells", 1, 1), ("one2all", 3, 2), ("one2one", 5, 2),
                                              ("opt_one2one", 5, 3)])
def test_policies_fake_multi_gpu_identical(xd, policy, n_ranks, c):
    """Logical GPUs = streams on device 0 (no kernel waits on another); results must be
    identical for every policy and device count, and no device runs two turns at once."""
    from synth import workload as W
    w = W.config("cfg1")
    with xd.Aligner(devices=[0, 0, 0], policy=policy, n_ranks=n_ranks, batch_size=37, subbatches=c) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        tr = al.trace()
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, policy)
    assert tr["n_pairs"].sum() == w.n_pairs
    for g in range(3):
        ev = np.sort(tr[tr["gpu"] == g], order="t0_ms")
        assert np.all(ev["t0_ms"][1:] >= ev["t1_ms"][:-1]), f"overlapping turns on gpu {g}"


def test_device_api_torch_tensors(xd):
    import torch
    from synth import workload as W
    w = W.config("cfg1")
    dev = torch.device("cuda:0")
    seq = torch.from_numpy(w.seq).to(dev)
    off = torch.from_numpy(w.offsets).to(dev)
    pairs = torch.from_numpy(w.pairs).to(dev)
    out = torch.zeros((w.n_pairs, 5), dtype=torch.int32, device=dev)
    cells = torch.zeros(w.n_pairs, dtype=torch.int64, device=dev)
    with xd.Aligner() as al:
        al.align_device(seq, off, pairs, out, cells, k=w.k, X=w.X, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    ref, rcells = oracle_of(w)
    o = out.cpu().numpy()
    for t, f in enumerate(FIELDS):
        assert np.array_equal(o[:, t], ref[f]), f
    assert np.array_equal(cells.cpu().numpy(), rcells)


def test_errors(xd):
    from synth import workload as W
    w = W.config("tiny")
    with xd.Aligner() as al:
        bad = w.seq.copy()
        bad[5] = ord("N")
        with pytest.raises(xd.XdropError) as e:
            al.align(bad, w.offsets, w.pairs, k=w.k, X=w.X)
        assert e.value.status == -4 and e.value.index == 5
        p = w.pairs.copy()
        p[3, 2] = 10 ** 6
        with pytest.raises(xd.XdropError) as e:
            al.align(w.seq, w.offsets, p, k=w.k, X=w.X)
        assert e.value.status == -5 and e.value.index == 3
        with pytest.raises(xd.XdropError):
            al.align(w.seq, w.offsets, w.pairs, k=0, X=w.X)
        with pytest.raises(xd.XdropError):
            al.align(w.seq, w.offsets, w.pairs, k=17, X=-1)
        r, c = al.align(w.seq, w.offsets, w.pairs[:0], k=w.k, X=w.X)
        assert r.shape == (0,)
        # still usable after errors
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, "after errors")


def test_lowercase_and_k31(xd):
    from synth import workload as W
    w = W.random_pairs_workload(seed=31, n_pairs=80, len_lo=40, len_hi=600, k=31, X=15)
    low = w.seq.copy()
    low[::3] = np.char.lower(low[::3].view("S1")).view(np.uint8)
    with xd.Aligner() as al:
        res, cells = al.align(low, w.offsets, w.pairs, k=31, X=15)
    ref, rcells = oracle_of(w, X=15)
    assert_same(res, cells, ref, rcells, "lowercase k31")


@pytest.mark.parametrize("long_g", ["0", "2", "4"])
@pytest.mark.parametrize("X", [0, 7, 15, 40])
def test_long_mode_multilane(xd, long_g, X, monkeypatch):
    """Every extension through the multi-lane long mode (alpha tiny) or none (G=0)."""
    from synth import workload as W
    monkeypatch.setenv("XDROP_LONG_G", long_g)
    monkeypatch.setenv("XDROP_LONG_ALPHA", "0.0001")
    w = W.random_pairs_workload(seed=300 + X, n_pairs=120, len_lo=0, len_hi=1500, k=13, X=X)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
        st = al.stats()
    ref, rcells = oracle_of(w, X=X)
    assert_same(res, cells, ref, rcells, f"long G={long_g} X={X}")
    if long_g != "0":
        assert st["long_items"] > 0


@pytest.mark.parametrize("X", [0, 5, 15, 60])
def test_reverse_complement_pairs(xd, X):
    """Strand (f2): XDROP_PAIR_RC pairs, mixed with forward pairs, every tier."""
    from synth import workload as W
    w = W.random_pairs_workload(seed=400 + X, n_pairs=160, len_lo=0, len_hi=1500, k=13, X=X, rc_frac=0.5)
    assert (w.pairs[:, 1] < 0).sum() > 40
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
    ref, rcells = oracle_of(w, X=X)
    assert_same(res, cells, ref, rcells, f"rc X={X}")


def test_reverse_complement_pool_workload(xd):
    from synth import workload as W
    w = W.make_pool_workload("rc-pool", 77, 300_000, 400, W._normal_len(3000, 400, 1000, 6000), 10.0, 500,
                             k=17, X=15, rc_frac=0.5, f_sp=0.05)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=17, X=15)
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, "rc pool")


def test_maximum_sizes_and_extreme_scoring(xd):
    """Reads at XDROP_MAX_READ_LEN (2^18), seed near both ends and the middle, k = 1024, and the
    largest scores the key range admits (M = 32 over 2^18 bases)."""
    from synth import workload as W
    rng = np.random.default_rng(5)
    L = 1 << 18
    a = rng.integers(0, 4, size=L, dtype=np.uint8)
    b = a.copy()
    mut = rng.random(L) < 0.02
    b[mut] = (b[mut] + 1) % 4
    seq = W.ASCII[np.concatenate([a, b])]
    off = np.array([0, L, 2 * L], np.int64)
    pairs = np.array([[0, 1, 0, 0], [0, 1, L - 1024, L - 1024], [0, 1, L // 2, L // 2],
                      [1, 0, 12345, 12345], [0, 0, L // 3, L // 3]], np.int32)   # last: identical read,
    # score M * 2^18 = 8.4M at M = 32 -- the top of the key range
    with xd.Aligner() as al:
        for (k, M, mu, g, X) in [(1024, 1, -1, -1, 15), (17, 32, -64, -64, 40), (31, 2, -3, -2, 0)]:
            p = pairs.copy()
            p[:, 2:] = np.minimum(p[:, 2:], L - k)
            if k == 1024:
                seq2 = seq.copy()                     # exact 1024-mer seeds
                for aa, bb, pa, pb in p:
                    seq2[off[bb] + pb: off[bb] + pb + k] = seq2[off[aa] + pa: off[aa] + pa + k]
            else:
                seq2 = seq
            res, cells = al.align(seq2, off, p, k=k, X=X, M=M, mu=mu, g=g)
            w2 = W.Workload("max", seq2, off, p, k, X, M, mu, g)
            ref, rcells = oracle_of(w2)
            assert_same(res, cells, ref, rcells, f"max k={k} M={M}")


def test_length_limit_error(xd):
    seq = np.frombuffer(b"A" * ((1 << 18) + 1), np.uint8)
    off = np.array([0, (1 << 18) + 1], np.int64)
    with xd.Aligner() as al:
        with pytest.raises(xd.XdropError) as e:
            al.align(seq, off, np.array([[0, 0, 0, 0]], np.int32), k=5, X=5)
        assert e.value.status == -6


@pytest.mark.parametrize("steal_min", ["0", "16", "200"])
def test_tail_stealing_resumes_exactly(xd, steal_min, monkeypatch):
    """Lane-mode extensions checkpointed at the tail and resumed 4 lanes wide stay exact."""
    from synth import workload as W
    monkeypatch.setenv("XDROP_STEAL_MIN", steal_min)
    monkeypatch.setenv("XDROP_LONG_G", "0")           # keep every extension in lane mode first
    w = W.random_pairs_workload(seed=77, n_pairs=300, len_lo=500, len_hi=4000, k=15, X=15, rc_frac=0.3)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, f"steal {steal_min}")
    if steal_min == "16":
        assert st["stolen"] > 0


def test_endgame_dispatch_exact(xd, monkeypatch):
    """The optional 4-lane endgame dispatch of T0 (XDROP_ENDGAME) stays exact."""
    from synth import workload as W
    monkeypatch.setenv("XDROP_ENDGAME", "100")        # every T0 batch in endgame mode
    w = W.random_pairs_workload(seed=78, n_pairs=200, len_lo=0, len_hi=2000, k=15, X=20, rc_frac=0.3)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, "endgame")


@pytest.mark.parametrize("M,mu,g,X", [(32, -64, -64, 478), (32, -64, -64, 479), (1, -1, -1, 509),
                                      (1, -1, -1, 510), (1, -4, -1, 15), (3, -9, -2, 40)])
def test_packed_range_gate_and_negative_mismatch(xd, M, mu, g, X):
    """The packed 16-bit T0 mode runs iff X + M <= 510; both sides of the gate, the
    API's extreme scores, and schemes whose offset-space mismatch score mu - 2g is negative (the
    borrow correction of the packed score word) stay exact."""
    from synth import workload as W
    w = W.random_pairs_workload(seed=600 + X + M, n_pairs=150, len_lo=0, len_hi=1200, k=13, X=X,
                                rc_frac=0.3)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X, M=M, mu=mu, g=g)
    ref, rcells = oracle_of(w, X=X, M=M, mu=mu, g=g)
    assert_same(res, cells, ref, rcells, f"gate M={M} mu={mu} g={g} X={X}")


@pytest.mark.parametrize("env", [{"XDROP_PK16": "0"}, {"XDROP_OCC": "1"},
                                 {"XDROP_T0_PER_SM": "1", "XDROP_IDLE_NS": "0"},
                                 {"XDROP_LONG_G": "2", "XDROP_LONG_ALPHA": "0.001"},
                                 {"XDROP_KERNEL": "1"}, {"XDROP_KERNEL": "2"},
                                 {"XDROP_KERNEL": "2", "XDROP_LONG_G": "2", "XDROP_LONG_ALPHA": "0.001"},
                                 {"XDROP_KERNEL": "2", "XDROP_OCC": "1", "XDROP_AGE_US": "0"},
                                 {"XDROP_KERNEL": "2", "XDROP_STEAL_MIN": "16", "XDROP_LONG_G": "0"},
                                 {"XDROP_KERNEL": "2", "XDROP_SHARED_T3": "0"}, {"XDROP_S1024": "1"}])
def test_kernel_variants_identical(xd, env, monkeypatch):
    """32-bit vs packed T0, 1 block/SM, 1 T0 block/SM (the rest escalation-only), packed 2-lane long
    mode, the tiered and the shared packed kernels (the shared one also with 2-lane
    long mode, one block per SM and immediate partial claims, and with tail stealing): every variant
    gives the oracle's results on an escalating, strand-mixed batch."""
    from synth import workload as W
    for k_, v in env.items():
        monkeypatch.setenv(k_, v)
    w = W.random_pairs_workload(seed=650, n_pairs=400, len_lo=0, len_hi=3000, k=13, X=25, rc_frac=0.4,
                                related=0.7)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, f"variant {env}")
    if env.get("XDROP_KERNEL") == "2":
        assert st["band_kernel"] == "shared"
        if env.get("XDROP_STEAL_MIN") == "16":       # a small batch idles most warps at once
            assert st["endgame_stolen"] > 0, st


@pytest.mark.parametrize("flags,env", [(8, "0"), (16, "0"), (8, "1"), (16, "1")])
def test_packed_resume_reaches_s1024(xd, flags, env, monkeypatch):
    """Unrelated continuations at X = 400 (packed path: X + M <= 510) outgrow T0 (32 cells), T1 (64
    tiered / 128 shared) and T2 (256): checkpoints resume in the packed 16-bit tiers up to the
    S = 1024 kernel, exactly, in both packed kernels."""
    from synth import workload as W
    monkeypatch.setenv("XDROP_S1024", env)            # 1: the S = 1024 level as a 4-warp CTA
    w = W.random_pairs_workload(seed=660, n_pairs=24, len_lo=2500, len_hi=4000, k=11, X=400, related=0.0)
    with xd.Aligner(flags=flags) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, f"packed resume S1024 flags={flags}")
    assert st["escalated"][2] > 0, st["escalated"]
    assert st["band_kernel"] == ("tiered" if flags == 8 else "shared")


@pytest.mark.parametrize("kernel", ["tiered", "shared"])
def test_packed_reaches_cta_levels(xd, kernel):
    """Unrelated continuations at X = 500 (still the packed path) outgrow S = 1024: the packed
    checkpoints resume in the 32-bit thread-block levels (S = 2048, then 4096), exactly."""
    from synth import workload as W
    w = W.random_pairs_workload(seed=661, n_pairs=12, len_lo=6000, len_hi=8000, k=11, X=500, related=0.0)
    with xd.Aligner(kernel=kernel) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, f"packed -> CTA {kernel}")
    assert st["band_kernel"] == kernel and st["cta_items"] > 0, st


def test_random_scoring_sweep_packed_and_32bit(xd):
    """40 random (M, mu, g, X) settings across the API ranges, both sides of the packed-mode gate,
    ragged strand-mixed batches: every field bit-exact against the oracle."""
    from synth import workload as W
    rng = np.random.default_rng(2024)
    with xd.Aligner() as al:
        for case in range(40):
            M = int(rng.choice([1, 1, 2, 3, 5, 32]))
            mu = -int(rng.choice([1, 1, 2, 4, 9, 64]))
            g = -int(rng.choice([1, 1, 2, 3, 7, 64]))
            X = int(rng.choice([0, 3, 15, 40, 200, 509 - M, 600]))
            w = W.random_pairs_workload(seed=7000 + case, n_pairs=40, len_lo=0, len_hi=700, k=9, X=X,
                                        rc_frac=0.3)
            res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X, M=M, mu=mu, g=g)
            ref, rcells = oracle_of(w, X=X, M=M, mu=mu, g=g)
            assert_same(res, cells, ref, rcells, f"case {case}: M={M} mu={mu} g={g} X={X}")
