"""GPU parity of the candidate-pair filters against oracle/filters.py.

f2 (BELLA's adaptive threshold; formula: DESIGN.md reading Q12): keep flags from
xdrop_adaptive_filter_device on the GPU's alignment results vs the oracle's flags on the ORACLE's
own alignment scores (the two score arrays are bit-identical by the parity tests), plus synthetic
scores placed exactly at, just below and just above the fp64 threshold.
f4 (k-mer frequency band): seed k-mer counts and band flags, bit-exact, on pools
with planted repeats (counts well inside and outside [20, 30]), reverse-complement copies, N bases
and k = 17 / 31."""
import math

import numpy as np
import pytest

from test_gpu_parity import oracle_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2309_07270_b200 as xd
    return xd


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def test_adaptive_filter_on_alignments(xd):
    import torch
    from oracle import filters as F
    from synth import workload as W
    w = W.config("ecoli", scale=0.1)
    ref, _ = oracle_of(w)
    seq, off, pairs = _dev(w.seq), _dev(w.offsets), _dev(w.pairs)
    out = torch.zeros((w.n_pairs, 5), dtype=torch.int32, device="cuda:0")
    with xd.Aligner(devices=[0]) as al:
        al.align_device(seq, off, pairs, out, None, k=w.k, X=w.X)
    # phi around the batch's own score-per-overlap-base quantiles, so that both outcomes occur
    ov = np.array([F.overlap_estimate(w.offsets, w.offsets, q) for q in w.pairs], dtype=np.float64)
    ratio = ref["score"] / np.maximum(ov, 1.0)
    mixed = 0
    for q, c in ((0.5, 8.0), (0.25, 0.0), (0.75, 20.0), (0.1, 2 * math.log(1e4))):
        phi = float(np.quantile(ratio, q))
        keep = torch.full((w.n_pairs,), 7, dtype=torch.uint8, device="cuda:0")
        xd.adaptive_filter_device(off, pairs, out, keep, phi, c)
        want = F.adaptive_keep(w.offsets, w.offsets, w.pairs, ref["score"], phi, c)
        got = keep.cpu().numpy()
        assert np.array_equal(got, want), (phi, c, np.nonzero(got != want)[0][:10])
        mixed += int(0 < want.sum() < w.n_pairs)
    assert mixed >= 2          # the quantile-placed thresholds split the batch


def test_adaptive_filter_threshold_boundary(xd):
    """Scores at floor/ceil of the fp64 threshold and at exact integer thresholds."""
    import torch
    from oracle import filters as F
    rng = np.random.default_rng(5)
    L = rng.integers(100, 5000, size=50)
    off = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)
    n = 4000
    a = rng.integers(0, 50, size=n); b = rng.integers(0, 50, size=n)
    pairs = np.stack([a, b, (rng.random(n) * L[a]).astype(int), (rng.random(n) * L[b]).astype(int)],
                     axis=1).astype(np.int32)
    phi, c = 0.5, 1.6
    t = np.array([phi * F.overlap_estimate(off, off, q) - math.sqrt(c * phi * F.overlap_estimate(off, off, q))
                  for q in pairs])
    scores = (np.floor(t) + rng.integers(-1, 3, size=n)).astype(np.int32)
    res = np.zeros((n, 5), dtype=np.int32)
    res[:, 0] = scores
    keep = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    xd.adaptive_filter_device(_dev(off), _dev(pairs), _dev(res), keep, phi, c)
    want = F.adaptive_keep(off, off, pairs, scores, phi, c)
    assert np.array_equal(keep.cpu().numpy(), want)
    assert 0 < want.sum() < n


def _pool_with_repeats(seed, n_reads, k, rc=True):
    """Random reads with planted k-mers repeated 1..60 times (some reverse-complemented) and a few N."""
    rng = np.random.default_rng(seed)
    reads = [list(rng.choice(list("ACGT"), size=int(rng.integers(k, 400)))) for _ in range(n_reads)]
    comp = {"A": "T", "C": "G", "G": "C", "T": "A"}
    planted = []
    for t in range(12):
        km = list(rng.choice(list("ACGT"), size=k))
        times = int([1, 5, 19, 20, 25, 30, 31, 45, 60, 2, 3, 27][t])
        for _ in range(times):
            r = int(rng.integers(0, n_reads))
            if len(reads[r]) < k:
                continue
            x = int(rng.integers(0, len(reads[r]) - k + 1))
            src = [comp[ch] for ch in reversed(km)] if (rc and rng.random() < 0.4) else km
            reads[r][x:x + k] = src
            planted.append((r, x))
    for _ in range(20):                                            # N bases (never inside a seed below)
        r = int(rng.integers(0, n_reads)); reads[r][int(rng.integers(0, len(reads[r])))] = "N"
    text = ["".join(r) for r in reads]
    seq = np.frombuffer("".join(text).encode(), dtype=np.uint8)
    off = np.concatenate([[0], np.cumsum([len(r) for r in text])]).astype(np.int64)
    pairs = []
    for (r, x) in planted + [(int(rng.integers(0, n_reads)), 0) for _ in range(200)]:
        if x + k <= len(text[r]) and "N" not in text[r][x:x + k]:
            pairs.append((r, 0, x, 0))
    return seq, off, np.array(pairs, dtype=np.int32)


@pytest.mark.parametrize("k", [17, 31, 5])
def test_seed_kmer_freq_parity(xd, k):
    import torch
    from oracle import filters as F
    seq, off, pairs = _pool_with_repeats(100 + k, 600, k)
    freq = torch.full((pairs.shape[0],), -1, dtype=torch.int32, device="cuda:0")
    keep = torch.full((pairs.shape[0],), 7, dtype=torch.uint8, device="cuda:0")
    xd.seed_kmer_freq_device(_dev(seq), _dev(off), _dev(pairs), k, 20, 30, freq=freq, keep=keep)
    wf, wk = F.seed_kmer_freq(seq, off, pairs, k, 20, 30)
    assert np.array_equal(freq.cpu().numpy(), wf)
    assert np.array_equal(keep.cpu().numpy(), wk)
    if k >= 17:
        assert wk.sum() > 0 and (wf > 30).any() and (wf < 20).any()


def test_seed_kmer_freq_errors(xd):
    import torch
    seq, off, pairs = _pool_with_repeats(7, 50, 17)
    bad = pairs.copy()
    bad[3, 2] = 10 ** 6
    freq = torch.zeros(pairs.shape[0], dtype=torch.int32, device="cuda:0")
    with pytest.raises(xd.XdropError) as e:
        xd.seed_kmer_freq_device(_dev(seq), _dev(off), _dev(bad), 17, 20, 30, freq=freq)
    assert e.value.status == -5 and e.value.index == 3
