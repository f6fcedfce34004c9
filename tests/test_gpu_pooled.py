"""Registered read pools (xdrop_pool_register / xdrop_align_pooled, include/xdrop.h):
the pool is uploaded and 2-bit packed once, then several batches (batches of 10,000)
are aligned against it moving only pairs and results.  Results must equal the oracle's and the
per-call host API's, for one device and for several logical devices under every policy (packed
words copied device-to-device), and registration must report bad bases and bad ids."""
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


def test_pooled_batches_match_oracle(xd):
    from synth import workload as W
    w = W.config("ecoli", scale=0.05)
    ref, rcells = oracle_of(w)
    with xd.Aligner() as al:
        pid = al.register_pool(w.seq, w.offsets)
        for lo in range(0, w.n_pairs, 1000):                  # batches against the resident pool
            hi = min(w.n_pairs, lo + 1000)
            res, cells = al.align_pooled(pid, w.pairs[lo:hi], k=w.k, X=w.X)
            assert_same(res, cells, ref[lo:hi], rcells[lo:hi], f"pooled batch {lo}")
        al.release_pool(pid)
        with pytest.raises(xd.XdropError):
            al.align_pooled(pid, w.pairs[:10], k=w.k, X=w.X)


@pytest.mark.parametrize("policy,n_ranks,c", [("cells", 1, 1), ("one2all", 3, 2), ("opt_one2one", 4, 1)])
def test_pooled_multi_device_policies(xd, policy, n_ranks, c):
    """Three logical devices (streams of device 0): the packed pool reaches slots 1, 2 by
    cudaMemcpyPeer; every policy gives the oracle's results."""
    from synth import workload as W
    w = W.config("cfg1")
    ref, rcells = oracle_of(w)
    with xd.Aligner(devices=[0, 0, 0], policy=policy, n_ranks=n_ranks, batch_size=37, subbatches=c) as al:
        pid = al.register_pool(w.seq, w.offsets)
        res, cells = al.align_pooled(pid, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    assert_same(res, cells, ref, rcells, f"pooled {policy}")
    assert st["cells"] == int(rcells.sum())          # stats summed over the devices and turns


def test_pooled_two_pools_and_errors(xd):
    from synth import workload as W
    w = W.random_pairs_workload(seed=91, n_pairs=120, len_lo=50, len_hi=1500, k=13, X=20, rc_frac=0.3)
    ref, rcells = oracle_of(w)
    with xd.Aligner() as al:
        pa = al.register_pool(w.seq, w.offsets)
        pb = al.register_pool(w.seq.copy(), w.offsets.copy())  # the same reads as a second pool (B side)
        res, cells = al.align_pooled(pa, w.pairs, k=w.k, X=w.X, pool_b=pb)
        assert_same(res, cells, ref, rcells, "two pools")
        bad = w.pairs.copy()
        bad[7, 3] = 1 << 20                                    # seed past the end of B
        with pytest.raises(xd.XdropError) as e:
            al.align_pooled(pa, bad, k=w.k, X=w.X, pool_b=pb)
        assert e.value.status == -5 and e.value.index == 7
        seq = w.seq.copy()
        seq[5] = ord("N")
        with pytest.raises(xd.XdropError) as e:
            al.register_pool(seq, w.offsets)
        assert e.value.status == -4 and e.value.index == 5
        res2, _ = al.align_pooled(pa, w.pairs, k=w.k, X=w.X)   # still usable after the errors
        assert np.array_equal(res2, ref)


def test_pooled_edge_cases(xd):
    """Empty batches and pools with empty reads; k-mer band and adaptive filter on empty inputs."""
    import torch
    from synth import workload as W
    w = W.random_pairs_workload(seed=93, n_pairs=40, len_lo=0, len_hi=400, k=9, X=10)
    ref, rcells = oracle_of(w)
    with xd.Aligner() as al:
        pid = al.register_pool(w.seq, w.offsets)
        res, cells = al.align_pooled(pid, w.pairs[:0], k=w.k, X=w.X)
        assert res.shape == (0,) and cells.shape == (0,)
        res, cells = al.align_pooled(pid, w.pairs, k=w.k, X=w.X)
        assert_same(res, cells, ref, rcells, "pool with empty reads")
        empty = al.register_pool(np.zeros(0, np.uint8), np.zeros(1, np.int64))
        res, _ = al.align_pooled(empty, w.pairs[:0], k=w.k, X=w.X)
        assert res.shape == (0,)
    dev = "cuda:0"
    z = torch.zeros((0, 4), dtype=torch.int32, device=dev)
    xd.seed_kmer_freq_device(torch.from_numpy(w.seq).to(dev), torch.from_numpy(w.offsets).to(dev), z, 17, 1, 5,
                             freq=torch.zeros(0, dtype=torch.int32, device=dev))
    xd.adaptive_filter_device(torch.from_numpy(w.offsets).to(dev), z, torch.zeros((0, 5), dtype=torch.int32, device=dev),
                              torch.zeros(0, dtype=torch.uint8, device=dev), 0.5, 1.0)
