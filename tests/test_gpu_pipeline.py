"""xd.Pipeline (several host-API batches in flight on one GPU, one context and host thread each):
every batch's results equal the serial call's and the oracle's, in submission order."""
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


def test_pipeline_matches_serial_and_oracle(xd):
    import oracle
    from synth import workload as W
    jobs, ws = [], []
    for t, X in enumerate([15, 0, 50, 15, 100, 5, 15]):
        w = W.random_pairs_workload(seed=1200 + t, n_pairs=150, len_lo=0, len_hi=2500, k=13, X=X, rc_frac=0.3)
        ws.append(w)
        jobs.append(dict(seqA=w.seq, offA=w.offsets, pairs=w.pairs, k=w.k, X=X))
    with xd.Pipeline(n_inflight=3) as pl:
        outs = pl.map(jobs)
        fut = pl.submit(**jobs[0])
        r0, c0 = fut.result()
    with xd.Aligner() as al:
        for (res, cells), job, w in zip(outs, jobs, ws):
            r, c = al.align(**job)
            assert all(np.array_equal(res[f], r[f]) for f in FIELDS) and np.array_equal(cells, c)
            ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs, w.k, X=job["X"])
            assert all(np.array_equal(res[f], ref[f]) for f in FIELDS) and np.array_equal(cells, rc)
    assert all(np.array_equal(r0[f], outs[0][0][f]) for f in FIELDS) and np.array_equal(c0, outs[0][1])


def test_pipeline_ecoli_batches(xd):
    """Whole E. coli-shaped batches, three in flight: identical to the serial call."""
    from synth import workload as W
    w = W.config("ecoli", scale=0.2)
    job = dict(seqA=w.seq, offA=w.offsets, pairs=w.pairs, k=w.k, X=w.X)
    with xd.Aligner() as al:
        r, c = al.align(**job)
    with xd.Pipeline(n_inflight=3) as pl:
        for res, cells in pl.map([job] * 6):
            assert np.array_equal(res, r) and np.array_equal(cells, c)
