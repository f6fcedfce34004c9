"""GPU parity on BASELINE.json configs 4 (X sweep, wide bands, spurious pairs) and 5
(C. elegans-shaped skewed lengths), at sizes the oracle finishes in seconds, plus
sampled parity on the full-size X-sweep batch in the launch configuration of the
bench tool (tools/configs_bench.py)."""
import numpy as np
import pytest

from test_gpu_parity import assert_same, oracle_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2309_07270_b200 as xd
    return xd


@pytest.fixture(scope="module")
def xsweep_small():
    from synth import workload as W
    # config 4 recipe (20 kb reads, f_sp = 0.2) with a short genome and 60 pairs
    return W.make_pool_workload("xsweep-small", 44, 400_000, 60, W._normal_len(20_000, 1_000, 19_000, 21_000),
                                6.0, 5_000, k=17, X=15, f_sp=0.2)


@pytest.mark.parametrize("flags", [8, 16])
@pytest.mark.parametrize("X", [15, 50, 100])
def test_xsweep_small_all_pairs(xd, xsweep_small, X, flags):
    """Both packed band kernels (tiered / shared)."""
    w = xsweep_small.with_X(X)
    with xd.Aligner(flags=flags) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=X)
        st = al.stats()
    ref, rcells = oracle_of(w, X=X)
    assert_same(res, cells, ref, rcells, f"xsweep X={X}")
    if X >= 50:
        assert st["escalated"][0] > 0          # the wide (warp-per-extension) levels ran


def test_xsweep_full_size_sampled(xd):
    """BASELINE configs[3] at full size (10k pairs of 20 kb): every 500th pair checked."""
    from synth import workload as W
    w = W.config("xsweep", X=50)
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=50)
    idx = np.arange(0, w.n_pairs, 500)
    ref, rcells = oracle_of(w, pairs=w.pairs[idx], X=50)
    assert_same(res[idx], cells[idx], ref, rcells, "xsweep full sampled")


@pytest.mark.parametrize("kernel", ["auto", "tiered", "shared"])
def test_celegans_shaped_small(xd, kernel):
    """BASELINE configs[4] recipe (lognormal 2-40 kb, f_sp = 0.1) at 1/2000 scale, per-call kernel
    choice and both packed kernels forced."""
    from synth import workload as W
    w = W.make_pool_workload("celegans-small", 55, 600_000, 400, W._lognormal_len(8_000, 0.6, 2_000, 40_000),
                             8.0, 1_000, k=17, X=15, f_sp=0.1)
    with xd.Aligner(kernel=kernel) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=15)
        st = al.stats()
    ref, rcells = oracle_of(w)
    assert_same(res, cells, ref, rcells, f"celegans small kernel={kernel}")
    # auto: 800 extensions cannot reach the probe threshold (1024 predicted escalations) -> tiered
    assert st["band_kernel"] == ("tiered" if kernel == "auto" else kernel)


def test_celegans_scaled_sample_shared_kernel_chosen(xd):
    """Config 5 at 1/20 scale (200k pairs): the per-batch probe predicts more than kSharedT1 = 1024
    T0 -> T1 checkpoints, so already the FIRST call runs the shared kernel; a stratified sample (every
    400th pair plus the 100 with the longest extensions) is bit-exact against the oracle, and both
    calls agree."""
    from synth import workload as W
    w = W.config("celegans", scale=0.05)
    with xd.Aligner() as al:
        r1, c1 = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        k1 = al.stats()["band_kernel"]
        r2, c2 = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
    assert k1 == "shared"
    assert st["escalated"][0] >= 1024 and st["band_kernel"] == "shared", (st["escalated"], st["band_kernel"])
    assert st["probe_overflows"] > 0
    L = np.diff(w.offsets)
    la, lb = L[w.pairs[:, 0]], L[w.pairs[:, 1] & 0x7fffffff]
    ext = np.minimum(w.pairs[:, 2], w.pairs[:, 3]) + np.minimum(la - w.pairs[:, 2], lb - w.pairs[:, 3])
    idx = np.unique(np.concatenate([np.arange(0, w.n_pairs, 400), np.argsort(-ext)[:100]]))
    ref, rcells = oracle_of(w, pairs=w.pairs[idx])
    assert_same(r2[idx], c2[idx], ref, rcells, "celegans x0.05 sampled")
