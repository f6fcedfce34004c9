"""GPU parity on EVERY pair of BASELINE.json configs 2 and 4 (config 1: test_gpu_parity.test_cfg1_full).

SURVEY.md §8(d): "Configs 1-4: every pair is checked".  The CUDA path runs in the bench's launch
configuration (xdrop_align_batch_device on HBM-resident tensors, the per-call kernel choice of a
warm context) and all five result fields plus the cell count of every pair are compared with the
CPU oracle (oracle/xdrop_oracle.c on all host threads).  Semantics every config must reproduce:
PAPER.md:224 (§IV-A, ``--ga 15``) and PAPER.md:87 (§II, anti-diagonal cells independent).
"""
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


def run_device(xd, w, calls=2):
    """The bench's step: device API on resident tensors; the last of `calls` calls is returned
    (a warm context makes the per-call kernel choice the bench's)."""
    import torch
    dev = torch.device("cuda:0")
    seq = torch.from_numpy(w.seq).to(dev)
    off = torch.from_numpy(w.offsets).to(dev)
    pairs = torch.from_numpy(w.pairs).to(dev)
    out = torch.full((w.n_pairs, 5), -7, dtype=torch.int32, device=dev)
    cells = torch.full((w.n_pairs,), -7, dtype=torch.int64, device=dev)
    kernels = []
    with xd.Aligner(devices=[0]) as al:
        for _ in range(calls):
            out.fill_(-7)
            cells.fill_(-7)
            al.align_device(seq, off, pairs, out, cells, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)
            kernels.append(al.stats()["band_kernel"])
    torch.cuda.synchronize(dev)
    o = out.cpu().numpy()
    res = np.zeros(w.n_pairs, dtype=xd.RESULT_DTYPE)
    for i, f in enumerate(("score", "a_begin", "a_end", "b_begin", "b_end")):
        res[f] = o[:, i]
    return res, cells.cpu().numpy(), kernels


@pytest.fixture(scope="module")
def ecoli():
    from synth import workload as W
    w = W.config("ecoli")
    ref, rcells = oracle_of(w)
    return w, ref, rcells


def test_ecoli_every_pair(xd, ecoli):
    """BASELINE configs[1] (the benched batch): all 100,000 pairs, bit-exact."""
    w, ref, rcells = ecoli
    res, cells, kernels = run_device(xd, w)
    assert_same(res, cells, ref, rcells, f"ecoli all pairs ({kernels})")
    assert int(cells.sum()) == int(rcells.sum())
    assert kernels == ["tiered", "tiered"]      # the probe predicts few escalations (no spurious pairs)


@pytest.fixture(scope="module")
def xsweep():
    from synth import workload as W
    return W.config("xsweep")


@pytest.mark.parametrize("X", [15, 50, 100])
def test_xsweep_every_pair(xd, xsweep, X):
    """BASELINE configs[3]: all 10,000 pairs of 20 kb reads at X = 15 / 50 / 100, bit-exact."""
    w = xsweep.with_X(X)
    res, cells, kernels = run_device(xd, w)
    ref, rcells = oracle_of(w, X=X)
    assert_same(res, cells, ref, rcells, f"xsweep X={X} all pairs ({kernels})")
    assert kernels == ["shared", "shared"]      # 20% spurious pairs (and every band at X >= 50) escalate


def test_ecoli_every_pair_host_api(xd, ecoli):
    """The same batch through the host API (xdrop_align_batch, the e2e leg of bench.py)."""
    w, ref, rcells = ecoli
    with xd.Aligner() as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
    assert_same(res, cells, ref, rcells, "ecoli all pairs, host API")


@pytest.mark.parametrize("policy,c", [("one2all", 1), ("one2one", 1), ("opt_one2one", 1), ("one2one", 4)])
def test_ecoli_every_pair_paper_policies(xd, ecoli, policy, c):
    """BASELINE configs[2]: the same E. coli-shaped batch under the paper's policies with its 16 ranks
    (PAPER.md:277), batches of 10,000 and c sub-batches, on four logical devices
    (streams of the one B200 here): every pair bit-exact, whatever the policy."""
    w, ref, rcells = ecoli
    with xd.Aligner(devices=[0, 0, 0, 0], policy=policy, n_ranks=16, batch_size=10000, subbatches=c) as al:
        res, cells = al.align(w.seq, w.offsets, w.pairs, k=w.k, X=w.X)
        st = al.stats()
    assert_same(res, cells, ref, rcells, f"ecoli {policy} c={c}")
    assert st["cells"] == int(rcells.sum())
