"""f4: several seeds per candidate pair, keep the best (reading Q26).

CPU: the oracle's selection pinned on hand-made cases and by brute force on tiny random inputs.
GPU: xdrop_align_multiseed / xdrop_best_seed_device against the oracle, element by element.
"""
import itertools

import numpy as np
import pytest

import oracle

RC = np.int32(-2 ** 31)


def test_best_seed_hand_cases():
    pairs = np.array([[0, 1, 5, 5], [0, 1, 9, 9], [0, 1, 20, 20], [2, 3, 0, 0], [0, 1, 7, 7],
                      [0, 1 | int(RC) & 0xffffffff, 3, 3]], dtype=np.int64).astype(np.int32)
    scores = np.array([5, 7, 7, 1, 9, 9])
    # rows 0-2 one candidate (max 7 first at row 1); row 3 alone; row 4 a separate candidate
    # (non-adjacent repeat); row 5 differs in the strand bit
    assert oracle.best_seed(pairs, scores).tolist() == [1, 1, 1, 3, 4, 5]
    assert oracle.best_seed(pairs[:0], scores[:0]).tolist() == []


def test_best_seed_brute_force():
    rng = np.random.default_rng(3)
    for n in range(1, 7):
        for _ in range(200):
            ids = rng.integers(0, 2, size=n)
            pairs = np.stack([ids, np.zeros(n, int), np.zeros(n, int), np.zeros(n, int)], 1).astype(np.int32)
            scores = rng.integers(-2, 3, size=n)
            got = oracle.best_seed(pairs, scores)
            for i in range(n):
                lo = i
                while lo > 0 and ids[lo - 1] == ids[i]:
                    lo -= 1
                hi = i
                while hi + 1 < n and ids[hi + 1] == ids[i]:
                    hi += 1
                cands = [t for t in range(lo, hi + 1) if scores[t] == max(scores[lo:hi + 1])]
                assert got[i] == cands[0]


@pytest.mark.gpu
def test_align_multiseed_matches_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2309_07270_b200 as xd
    from synth import workload as W
    w = W.make_pool_workload("ms", 91, 200_000, 150, W._normal_len(2000, 300, 800, 4000), 8.0, 300,
                             k=15, X=15, rc_frac=0.3, seeds_per_pair=3, f_sp=0.1)
    ref, rcells = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, X=w.X)
    rbest = oracle.best_seed(w.pairs, ref["score"])
    with xd.Aligner() as al:
        res, best, cells = al.align_multiseed(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        assert np.array_equal(res, ref) and np.array_equal(cells, rcells)
        assert np.array_equal(best, rbest)
        # device form on torch tensors
        dev = torch.device("cuda:0")
        seq = torch.from_numpy(w.seq).to(dev)
        off = torch.from_numpy(w.offsets).to(dev)
        pr = torch.from_numpy(w.pairs.reshape(-1, 4).copy()).to(dev)
        out = torch.zeros((pr.shape[0], 5), dtype=torch.int32, device=dev)
        al.align_device(seq, off, pr, out, None, k=w.k, X=w.X)
        b = torch.zeros(pr.shape[0], dtype=torch.int64, device=dev)
        al.best_seed_device(pr, out, b)
        assert np.array_equal(b.cpu().numpy(), rbest)
        with pytest.raises(xd.XdropError):
            import ctypes
            from paper_2309_07270_b200 import _native as N
            N.check(N.lib.xdrop_best_seed_device(al._h, None, None, -1, None, None), "neg", al._h)
    assert (np.bincount(rbest) > 0).sum() < len(rbest)       # several seeds really shared candidates
