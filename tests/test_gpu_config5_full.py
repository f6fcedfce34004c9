"""BASELINE configs[4] at FULL size (5,000,000 C. elegans-shaped pairs, ~1e12 cells) in the bench's
launch configuration (device API, HBM-resident inputs): a stratified sample -- every 100th pair in cost
order plus the 1,000 longest -- bit-exact against the oracle (the second of two calls
of a context; the per-batch probe picks the shared kernel for both), plus properties on every pair."""
import numpy as np
import pytest

from test_gpu_full_parity import run_device
from test_gpu_parity import assert_same, oracle_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2309_07270_b200 as xd
    return xd


def test_config5_full_stratified(xd):
    from synth import workload as W
    w = W.config("celegans")
    assert w.n_pairs == 5_000_000
    res, cells, kernels = run_device(xd, w, calls=2)
    assert kernels == ["shared", "shared"]
    L = np.diff(w.offsets)
    p = w.pairs
    cost = np.minimum(p[:, 2], p[:, 3]) + np.minimum(L[p[:, 0]] - p[:, 2] - w.k, L[p[:, 1] & 0x7fffffff] - p[:, 3] - w.k)
    order = np.argsort(-cost, kind="stable")
    idx = np.unique(np.concatenate([order[::100], order[:1000]]))
    ref, rcells = oracle_of(w, pairs=p[idx])
    assert_same(res[idx], cells[idx], ref, rcells, "config 5 full, stratified sample")
    # properties at any size, on every pair
    assert np.all(res["a_begin"] <= p[:, 2]) and np.all(res["a_end"] >= p[:, 2] + w.k)
    assert np.all(cells >= 2)
