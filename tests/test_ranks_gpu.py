"""f1 on the GPU: OS-process ranks share the device under each policy's token ring; the
alignments (through the C ABI, device-resident pools) equal the single-process results and
the oracle, and the gathered trace passes the scheduler verifiers."""
import numpy as np
import pytest

from test_gpu_parity import oracle_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy,n_ranks,c", [("one2all", 3, 1), ("one2one", 4, 2), ("opt_one2one", 4, 2)])
def test_ranks_share_one_gpu(policy, n_ranks, c):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2309_07270_b200 import ranks as R
    from synth import workload as W
    w = W.config("cfg1")
    out, cells, turns, met, bad = R.spawn(n_ranks, policy, 1, w.seq, w.offsets, w.pairs, batch_size=23, c=c,
                                          params=dict(k=w.k, X=w.X), use_gpu=True, timeout=300)
    assert bad == [], bad
    ref, rcells = oracle_of(w)
    for t, f in enumerate(("score", "a_begin", "a_end", "b_begin", "b_end")):
        assert np.array_equal(out[:, t], ref[f]), f
    assert np.array_equal(cells, rcells)
    assert met["handoffs"] > 0
