"""Pins for the CPU oracle against things other than itself (-m "not gpu").

Each test names the pin from DESIGN.md §Pins / SURVEY.md §8(c):
  brute force  -- all alignment paths enumerated explicitly (definition of an
                  alignment score, no DP) pin FULLDP; FULLDP pins EXTEND when X
                  exceeds the no-pruning bound (P-1)
  closed forms -- identical strings (P-2), single substitution (P-3),
                  all-mismatch cell count (X+2)^2 (P-4), unpruned cell count
                  (m+1)(n+1)
  hand traces  -- tests/golden/extend_hand.txt
  invariants   -- upper bound (P-5), symmetry (P-6), achievability (P-7),
                  left/right mirror (P-8)
Both oracle implementations (C: oracle.extend, Python: xdrop_ref.extend) are
pinned by the same checks, and must agree with each other.
"""
import itertools

import numpy as np
import os
import random

import pytest

import oracle
from oracle import xdrop_ref as ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALPH = "ACGT"


def impls():
    return [("c", oracle.extend), ("py", ref.extend)]


# ----------------------------------------------------------------- brute force
def enumerate_best(a, b, M, mu, g):
    """Max score of every cell by explicit enumeration of all move sequences."""
    m, n = len(a), len(b)
    best = {}

    def walk(i, j, v):
        if best.get((i, j), None) is None or v > best[(i, j)]:
            best[(i, j)] = v
        if i < m and j < n:
            walk(i + 1, j + 1, v + (M if a[i] == b[j] else mu))
        if i < m:
            walk(i + 1, j, v + g)
        if j < n:
            walk(i, j + 1, v + g)

    walk(0, 0, 0)
    return best


def argmax_rule(cellvals):
    """Tie-break of reading Q8: smallest anti-diagonal, then smallest i."""
    top = max(cellvals.values())
    i, j = min(((i, j) for (i, j), v in cellvals.items() if v == top), key=lambda c: (c[0] + c[1], c[0]))
    return top, i, j


@pytest.mark.parametrize("M,mu,g", [(1, -1, -1), (2, -3, -2), (5, -4, -3)])
def test_fulldp_matches_path_enumeration(M, mu, g):
    rng = random.Random(7)
    for _ in range(120):
        a = "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 4)))
        b = "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 4)))
        assert ref.fulldp(a, b, M, mu, g) == argmax_rule(enumerate_best(a, b, M, mu, g))


def no_prune_bound(m, n, M, mu, g):
    # P-1: best <= min(m,n)*M and every H(i,j) >= -max(i,j)*max(-mu,-g)
    return min(m, n) * M + max(m, n) * max(-mu, -g)


def strings(alph, maxlen):
    for L in range(maxlen + 1):
        for t in itertools.product(alph, repeat=L):
            yield "".join(t)


@pytest.mark.parametrize("name,fn", impls())
def test_P1_exhaustive_tiny_equals_fulldp(name, fn):
    pool = list(strings("AC", 4)) + list(strings(ALPH, 2))
    for a in pool:
        for b in pool:
            X = no_prune_bound(len(a), len(b), 1, -1, -1)
            best, i, j, cells = fn(a, b, 1, -1, -1, X)
            assert (best, i, j) == ref.fulldp(a, b), (a, b)
            assert cells == (len(a) + 1) * (len(b) + 1), (a, b)  # nothing pruned -> full rectangle


@pytest.mark.parametrize("name,fn", impls())
@pytest.mark.parametrize("M,mu,g", [(1, -1, -1), (2, -3, -2), (5, -4, -3)])
def test_P1_random_equals_fulldp(name, fn, M, mu, g):
    rng = random.Random(11)
    for _ in range(60):
        a = "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 25)))
        b = list(a) if rng.random() < 0.5 else [rng.choice(ALPH) for _ in range(rng.randint(0, 25))]
        for t in range(len(b)):
            if rng.random() < 0.15:
                b[t] = rng.choice(ALPH)
        b = "".join(b)
        X = no_prune_bound(len(a), len(b), M, mu, g)
        best, i, j, cells = fn(a, b, M, mu, g, X)
        assert (best, i, j) == ref.fulldp(a, b, M, mu, g)
        assert cells == (len(a) + 1) * (len(b) + 1)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("name,fn", impls())
def test_P2_identical(name, fn):
    rng = random.Random(3)
    for L in [0, 1, 2, 7, 31, 64]:
        a = "".join(rng.choice(ALPH) for _ in range(L))
        for X in [0, 1, 5, 15, 100]:
            for (M, mu, g) in [(1, -1, -1), (2, -3, -2)]:
                best, i, j, _ = fn(a, a, M, mu, g, X)
                assert (best, i, j) == (L * M, L, L)


@pytest.mark.parametrize("name,fn", impls())
def test_P3_single_substitution(name, fn):
    rng = random.Random(5)
    for L in [4, 9, 20, 40]:
        a = "".join(rng.choice(ALPH) for _ in range(L))
        for p in range(0, L - 2):
            b = list(a)
            b[p] = ALPH[(ALPH.index(a[p]) + 1) % 4]
            b = "".join(b)
            assert fn(a, b, 1, -1, -1, 0)[:3] == (p, p, p)
            for X in [1, 2, 15]:
                assert fn(a, b, 1, -1, -1, X)[:3] == (L - 2, L, L), (a, b, p, X)


@pytest.mark.parametrize("name,fn", impls())
def test_P4_all_mismatch_cells(name, fn):
    for X in [0, 1, 2, 5, 15]:
        for extra in [0, 1, 7]:
            m, n = X + 1 + extra, X + 1 + (extra * 2) % 5
            assert fn("A" * m, "C" * n, 1, -1, -1, X) == (0, 0, 0, (X + 2) ** 2)


# ----------------------------------------------------------------- hand traces
def load_golden():
    rows = []
    with open(os.path.join(GOLDEN, "extend_hand.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            lhs, rhs = line.split("|")
            a, b, M, mu, g, X = lhs.split()
            a = "" if a == "-" else a
            b = "" if b == "-" else b
            rows.append((a, b, int(M), int(mu), int(g), int(X), tuple(int(t) for t in rhs.split())))
    return rows


@pytest.mark.parametrize("name,fn", impls())
def test_golden_hand_traces(name, fn):
    rows = load_golden()
    assert len(rows) >= 6
    for a, b, M, mu, g, X, want in rows:
        assert fn(a, b, M, mu, g, X) == want, (a, b, X)


# ------------------------------------------------------------------ invariants
def mutate(rng, a, err):
    out = []
    for ch in a:
        r = rng.random()
        if r < err / 3:
            continue                                    # deletion
        if r < 2 * err / 3:
            out.append(rng.choice(ALPH))                # insertion
        if r < err:
            out.append(ALPH[(ALPH.index(ch) + rng.randint(1, 3)) % 4])  # substitution
        else:
            out.append(ch)
    return "".join(out)


def test_invariants_P5_P6_P7_and_twins_agree():
    rng = random.Random(13)
    for _ in range(400):
        L = rng.randint(0, 30)
        a = "".join(rng.choice(ALPH) for _ in range(L))
        b = mutate(rng, a, 0.25) if rng.random() < 0.7 else "".join(
            rng.choice(ALPH) for _ in range(rng.randint(0, 30)))
        M, mu, g = rng.choice([(1, -1, -1), (2, -3, -2), (5, -4, -3), (2, -1, -1)])
        full = ref.fulldp(a, b, M, mu, g)
        for X in [0, 1, 2, 3, 5, 10]:
            c = oracle.extend(a, b, M, mu, g, X)
            p = ref.extend(a, b, M, mu, g, X)
            assert c == p, (a, b, X)                     # the two oracles agree
            assert c[0] <= full[0]                       # P-5 upper bound
            sw = oracle.extend(b, a, M, mu, g, X)
            assert sw[0] == c[0] and sw[3] == c[3]       # P-6 symmetry (score, cells)
            # P-7 achievability: the unpruned optimum at (i*, j*) is >= best
            assert ref.fulldp(a[:c[1]], b[:c[2]], M, mu, g) is not None
            sub = ref.fulldp(a[:c[1]], b[:c[2]], M, mu, g)
            # H_full(i*, j*) is the NW value of the prefixes: recompute directly
            assert nw(a[:c[1]], b[:c[2]], M, mu, g) >= c[0]
            assert sub[0] >= c[0]


def nw(a, b, M, mu, g):
    """Global NW score of a vs b via path enumeration on tiny, DP otherwise."""
    m, n = len(a), len(b)
    prev = [j * g for j in range(n + 1)]
    for i in range(1, m + 1):
        cur = [i * g] + [0] * n
        for j in range(1, n + 1):
            cur[j] = max(prev[j] + g, cur[j - 1] + g, prev[j - 1] + (M if a[i - 1] == b[j - 1] else mu))
        prev = cur
    return prev[n]


def test_P8_left_right_mirror_and_align_wiring():
    rng = random.Random(17)
    for _ in range(200):
        A = "".join(rng.choice(ALPH) for _ in range(rng.randint(5, 60)))
        B = mutate(rng, A, 0.2)
        k = rng.randint(1, 4)
        if len(B) < k:
            continue
        a_pos = rng.randint(0, len(A) - k)
        b_pos = rng.randint(0, len(B) - k)
        X = rng.choice([0, 2, 7, 15])
        r = oracle.align(A, B, a_pos, b_pos, k, 1, -1, -1, X)
        # mirror: left extension == right extension of the reversed reads at the mirrored seed
        rr = oracle.align(A[::-1], B[::-1], len(A) - a_pos - k, len(B) - b_pos - k, k, 1, -1, -1, X)
        assert r["left"] == rr["right"] and r["right"] == rr["left"]
        assert r["score"] == rr["score"] and r["cells"] == rr["cells"]
        assert (r["a_begin"], r["a_end"]) == (len(A) - rr["a_end"], len(A) - rr["a_begin"])
        # wiring against the pure-Python twin
        p = ref.align(A, B, a_pos, b_pos, k, 1, -1, -1, X)
        assert {kk: r[kk] for kk in p} == p


def test_align_identical_reads_closed_form():
    rng = random.Random(19)
    for _ in range(50):
        A = "".join(rng.choice(ALPH) for _ in range(rng.randint(20, 200)))
        k = 17 if len(A) >= 17 else 1
        pos = rng.randint(0, len(A) - k)
        for X in [0, 15]:
            r = oracle.align(A, A, pos, pos, k, 1, -1, -1, X)
            assert (r["score"], r["a_begin"], r["a_end"], r["b_begin"], r["b_end"]) == (len(A), 0, len(A), 0, len(A))


def test_survey_regression_nonmonotone_in_X():
    """SURVEY.md §0 finding 2 (two independent scratch implementations during the survey):
    the X-drop score is NOT monotone in X; our oracle must reproduce the printed triple."""
    a, b = "ATCACTGAGCATATGGTC", "CACTATTGAGCATCAGGGTC"
    got = {X: oracle.extend(a, b, 1, -1, -1, X)[:3] for X in (1, 2, 3)}
    assert got == {1: (9, 18, 20), 2: (2, 6, 4), 3: (9, 18, 20)}


def test_batch_matches_single():
    rng = random.Random(23)
    import numpy as np
    reads = ["".join(rng.choice(ALPH) for _ in range(rng.randint(30, 120))) for _ in range(12)]
    seq = np.frombuffer("".join(reads).encode(), dtype=np.uint8)
    off = np.zeros(len(reads) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(r) for r in reads])
    pairs = []
    for _ in range(40):
        ai, bi = rng.randrange(12), rng.randrange(12)
        pairs.append((ai, bi, rng.randint(0, len(reads[ai]) - 5), rng.randint(0, len(reads[bi]) - 5)))
    res, cells = oracle.align_batch(seq, off, seq, off, np.array(pairs), 5, X=7, nthreads=3)
    for t, (ai, bi, ap, bp) in enumerate(pairs):
        r = oracle.align(reads[ai], reads[bi], ap, bp, 5, X=7)
        assert (res[t]["score"], res[t]["a_begin"], res[t]["a_end"], res[t]["b_begin"],
                res[t]["b_end"], cells[t]) == (r["score"], r["a_begin"], r["a_end"],
                                                r["b_begin"], r["b_end"], r["cells"])


def test_batch_reports_bad_seed():
    import numpy as np
    seq = np.frombuffer(b"ACGTACGT", dtype=np.uint8)
    off = np.array([0, 8], dtype=np.int64)
    with pytest.raises(ValueError):
        oracle.align_batch(seq, off, seq, off, np.array([[0, 0, 5, 0]]), 5)


# ------------------------------------------------------------ strand (f2)
def _rc(s):
    return s.translate(str.maketrans("ACGT", "TGCA"))[::-1]


def test_rc_pairs_closed_form_and_equivalence():
    """Reading Q16: a pair with XDROP_PAIR_RC aligns A against revcomp(B), B coordinates in
    revcomp(B).  Pinned by (1) B = revcomp(A) behaving exactly like identical reads (closed
    form), (2) equality with the same pair written forward on an explicitly reverse-
    complemented pool (a different input path through the oracle)."""
    import numpy as np
    rng = random.Random(29)
    reads, pairs_rc, pairs_fw, fw_reads = [], [], [], []
    for p in range(40):
        A = "".join(rng.choice(ALPH) for _ in range(rng.randint(30, 150)))
        Bf = mutate(rng, A, 0.15) if p % 2 else A        # forward-strand partner
        if len(Bf) < 6:
            Bf = A
        pa = rng.randint(0, len(A) - 5)
        pb = rng.randint(0, len(Bf) - 5)
        Bs = _rc(Bf)                                     # stored on the other strand
        reads += [A, Bs]
        fw_reads += [A, Bf]
        pairs_rc.append((2 * p, (2 * p + 1) | -(1 << 31), pa, pb))
        pairs_fw.append((2 * p, 2 * p + 1, pa, pb))
        if p % 2 == 0:                                   # B = revcomp(A): identical after RC
            r = oracle.align_batch(np.frombuffer((A + Bs).encode(), np.uint8),
                                   np.array([0, len(A), len(A) + len(Bs)]), np.frombuffer((A + Bs).encode(), np.uint8),
                                   np.array([0, len(A), len(A) + len(Bs)]),
                                   np.array([[0, 1 | -(1 << 31), pa, pa]]), 5, X=7)[0][0]
            assert (r["score"], r["a_begin"], r["a_end"], r["b_begin"], r["b_end"]) == (len(A), 0, len(A), 0, len(A))

    def pool(rs):
        off = np.zeros(len(rs) + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in rs])
        return np.frombuffer("".join(rs).encode(), np.uint8), off
    s1, o1 = pool(reads)
    s2, o2 = pool(fw_reads)
    r1, c1 = oracle.align_batch(s1, o1, s1, o1, np.array(pairs_rc), 5, X=9)
    r2, c2 = oracle.align_batch(s2, o2, s2, o2, np.array(pairs_fw), 5, X=9)
    assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
    for t, (a, b, pa, pb) in enumerate(pairs_rc):         # and the Python twin
        p = ref.align(reads[a], reads[b & 0x7fffffff], pa, pb, 5, X=9, rc=True)
        assert (r1[t]["score"], r1[t]["b_begin"], r1[t]["b_end"], c1[t]) == (p["score"], p["b_begin"], p["b_end"], p["cells"])


# ----------------------------------------------------------- f2 / f4 filter oracles (oracle/filters.py)
def test_adaptive_keep_closed_form():
    """Reading Q12 by hand: |A| = 100, |B| = 80, a_pos = 30, b_pos = 10 -> ov = min(30, 10) +
    min(70, 70) = 80; phi = 0.5 -> mu = 40; c = 1.6 -> sqrt(64) = 8 -> threshold 32 (exact in
    binary), so score 32 is kept and 31 is not; c = 0 -> the threshold is mu itself; c = 1e9 puts it
    at 40 - 2e5, below every score here."""
    from oracle import filters as F
    off = np.array([0, 100, 180], dtype=np.int64)
    pairs = np.array([[0, 1, 30, 10]] * 4, dtype=np.int32)
    assert F.overlap_estimate(off, off, pairs[0]) == 80
    assert list(F.adaptive_keep(off, off, pairs, [32, 31, 40, 39], 0.5, 1.6)) == [1, 0, 1, 1]
    assert list(F.adaptive_keep(off, off, pairs, [40, 39, 41, 0], 0.5, 0.0)) == [1, 0, 1, 0]
    assert list(F.adaptive_keep(off, off, pairs, [0, 1, 5, -1], 0.5, 1e9)) == [1, 1, 1, 1]   # t = 40 - 2e5 < -1
    # the RC bit of b_id does not change B's length; seeds at the read ends give ov = the other side
    rc = np.array([[0, 1 | -(1 << 31), 0, 0], [0, 1, 100, 80]], dtype=np.int32)
    assert F.overlap_estimate(off, off, rc[0]) == 80 and F.overlap_estimate(off, off, rc[1]) == 80


def test_adaptive_keep_monotone():
    """keep is monotone in the score and antitone in phi (for c fixed), at any size."""
    from oracle import filters as F
    rng = np.random.default_rng(3)
    off = np.concatenate([[0], np.cumsum(rng.integers(200, 2000, size=20))]).astype(np.int64)
    L = np.diff(off)
    n = 300
    a = rng.integers(0, 20, size=n); b = rng.integers(0, 20, size=n)
    pairs = np.stack([a, b, (rng.random(n) * (L[a] - 17)).astype(int), (rng.random(n) * (L[b] - 17)).astype(int)],
                     axis=1).astype(np.int32)
    s = rng.integers(-50, 2000, size=n)
    k1 = F.adaptive_keep(off, off, pairs, s, 0.3, 8.0)
    assert np.all(F.adaptive_keep(off, off, pairs, s + 1, 0.3, 8.0) >= k1)
    assert np.all(F.adaptive_keep(off, off, pairs, s, 0.4, 8.0) <= k1)


def test_seed_kmer_freq_hand_cases():
    """Canonical k-mer counts by hand.  Pool ["AAAA", "TTTT", "ACG", "TAC", "ANAC"], k = 3:
    AAA occurs twice in read 0 and its reverse complement TTT twice in read 1 -> 4; ACG (its
    reverse complement CGT) occurs once in read 2 -- the CGT across the read-2/read-3 boundary does
    not count; TAC (canonical GTA) once in read 3; the 3-mers of read 4 with N do not count, NAC
    neither, so nothing else is added."""
    from oracle import filters as F
    reads = ["AAAA", "TTTT", "ACG", "TAC", "ANAC"]
    seq = np.frombuffer("".join(reads).encode(), dtype=np.uint8)
    off = np.concatenate([[0], np.cumsum([len(r) for r in reads])]).astype(np.int64)
    pairs = np.array([[0, 1, 0, 0], [1, 0, 1, 0], [2, 0, 0, 0], [3, 0, 0, 0]], dtype=np.int32)
    freq, keep = F.seed_kmer_freq(seq, off, pairs, 3, 2, 4)
    assert list(freq) == [4, 4, 1, 1] and list(keep) == [1, 1, 0, 0]
    assert F.canonical("ACG") == "ACG" and F.canonical("CGT") == "ACG" and F.canonical("TAC") == "GTA"
    assert F.canonical("ANA") is None
    counts = F.kmer_counts(seq, off, 3)
    assert counts == {"AAA": 4, "ACG": 1, "GTA": 1}


def test_seed_kmer_freq_invariants():
    """Every valid seed occurs at least once (itself); a seed and its reverse complement planted in
    another read have the same count; the counts sum to the number of ACGT k-mer positions."""
    from oracle import filters as F
    rng = np.random.default_rng(11)
    reads = ["".join(rng.choice(list("ACGT"), size=int(rng.integers(5, 60)))) for _ in range(30)]
    seq = np.frombuffer("".join(reads).encode(), dtype=np.uint8)
    off = np.concatenate([[0], np.cumsum([len(r) for r in reads])]).astype(np.int64)
    k = 4
    pairs = np.array([[r, 0, int(rng.integers(0, len(reads[r]) - k + 1)), 0] for r in range(30)], dtype=np.int32)
    freq, _ = F.seed_kmer_freq(seq, off, pairs, k, 0, 10 ** 9)
    assert np.all(freq >= 1)
    assert sum(F.kmer_counts(seq, off, k).values()) == sum(max(0, len(r) - k + 1) for r in reads)
    km = reads[0][:k]
    rcs = "".join({"A": "T", "C": "G", "G": "C", "T": "A"}[c] for c in reversed(km))
    reads2 = reads + [rcs]
    seq2 = np.frombuffer("".join(reads2).encode(), dtype=np.uint8)
    off2 = np.concatenate([[0], np.cumsum([len(r) for r in reads2])]).astype(np.int64)
    f0, _ = F.seed_kmer_freq(seq, off, np.array([[0, 0, 0, 0]], dtype=np.int32), k, 0, 99)
    f1, _ = F.seed_kmer_freq(seq2, off2, np.array([[0, 0, 0, 0], [30, 0, 0, 0]], dtype=np.int32), k, 0, 99)
    assert f1[0] == f1[1] == f0[0] + 1


# ------------------------------------------ SeqAn/LOGAN-style mode (f3, Q28-Q30)
def compat_impls():
    return [("c", lambda *a: oracle.extend(*a, compat=True)),
            ("py", lambda *a: ref.extend(*a, compat=True))]


@pytest.mark.parametrize("name,fn", compat_impls())
def test_compat_hand_traces(name, fn):
    rows = []
    with open(os.path.join(GOLDEN, "extend_compat_hand.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                lhs, rhs = line.split("|")
                a, b, M, mu, g, X = lhs.split()
                rows.append(("" if a == "-" else a, "" if b == "-" else b, int(M), int(mu), int(g), int(X),
                             tuple(int(t) for t in rhs.split())))
    assert len(rows) >= 6
    for a, b, M, mu, g, X, want in rows:
        assert fn(a, b, M, mu, g, X) == want, (a, b, X)


@pytest.mark.parametrize("name,fn", compat_impls())
def test_compat_unpruned_is_global_alignment(name, fn):
    """With X above the no-pruning bound (strictly, so the Q28 edge rule never bites) every cell
    lives, the last anti-diagonal is m+n, and the longest extension is the corner: (H(m,n), m, n)
    with H(m,n) the GLOBAL alignment score -- by brute-force path enumeration on tiny inputs."""
    pool = list(strings("AC", 3)) + list(strings(ALPH, 2))
    for (M, mu, g) in [(1, -1, -1), (2, -3, -2)]:
        for a in pool:
            for b in pool:
                X = no_prune_bound(len(a), len(b), M, mu, g) + 1
                glob = enumerate_best(a, b, M, mu, g)[(len(a), len(b))]
                assert fn(a, b, M, mu, g, X) == (glob, len(a), len(b), (len(a) + 1) * (len(b) + 1)), (a, b)


def nw_global(a, b, M, mu, g):
    """Textbook Needleman-Wunsch global score (row by row, whole table)."""
    prev = [j * g for j in range(len(b) + 1)]
    for i in range(1, len(a) + 1):
        cur = [i * g] + [0] * len(b)
        for j in range(1, len(b) + 1):
            cur[j] = max(prev[j - 1] + (M if a[i - 1] == b[j - 1] else mu), prev[j] + g, cur[j - 1] + g)
        prev = cur
    return prev[-1]


@pytest.mark.parametrize("name,fn", compat_impls())
def test_compat_unpruned_random_nw(name, fn):
    rng = random.Random(29)
    for _ in range(60):
        a = "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 20)))
        b = mutate(rng, a, 0.2) if rng.random() < 0.6 else "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 20)))
        for (M, mu, g) in [(1, -1, -1), (5, -4, -3)]:
            X = no_prune_bound(len(a), len(b), M, mu, g) + 1
            assert fn(a, b, M, mu, g, X) == (nw_global(a, b, M, mu, g), len(a), len(b),
                                             (len(a) + 1) * (len(b) + 1)), (a, b)


@pytest.mark.parametrize("name,fn", compat_impls())
def test_compat_closed_forms(name, fn):
    rng = random.Random(31)
    # identical strings: the diagonal reaches the corner for every X >= 0
    for L in [0, 1, 7, 31]:
        a = "".join(rng.choice(ALPH) for _ in range(L))
        for X in [0, 1, 15]:
            assert fn(a, a, 2, -3, -2, X)[:3] == (2 * L, L, L)
    # all mismatches, unit scoring, X >= 1: best stays 0, the boundary lives for j <= X-1 only (Q28),
    # the interior square [1..X]^2 lives (H = -max(i,j) >= -X), so the last live anti-diagonal is 2X
    # with the single cell (X,X), H = -X (Q29/Q30); computed cells: the live (X+1)^2 - 2, the two dead
    # boundary cells (0,X), (X,0), row X+1 (j = 1..X+1) and column X+1 (i = 1..X): (X+2)^2 - 2.
    for X in [1, 2, 5, 15]:
        for extra in [0, 1, 7]:
            m, n = X + 1 + extra, X + 1 + (extra * 2) % 5
            assert fn("A" * m, "C" * n, 1, -1, -1, X) == (-X, X, X, (X + 2) ** 2 - 2)
    # single substitution at p (unit scoring): X = 0 stops at (p,p); X >= 1 bridges it to the corner
    for L in [4, 9, 20]:
        a = "".join(rng.choice(ALPH) for _ in range(L))
        for p in range(0, L - 2):
            b = a[:p] + ALPH[(ALPH.index(a[p]) + 1) % 4] + a[p + 1:]
            assert fn(a, b, 1, -1, -1, 0)[:3] == (p, p, p)
            for X in [1, 2, 15]:
                assert fn(a, b, 1, -1, -1, X)[:3] == (L - 2, L, L)


def test_compat_twins_agree_and_align_wiring():
    rng = random.Random(37)
    for _ in range(300):
        a = "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 40)))
        b = mutate(rng, a, rng.choice([0.05, 0.15, 0.3])) if rng.random() < 0.8 else \
            "".join(rng.choice(ALPH) for _ in range(rng.randint(0, 40)))
        X = rng.choice([0, 1, 2, 5, 15])
        sc = rng.choice([(1, -1, -1), (2, -3, -2), (1, -2, -1)])
        got = oracle.extend(a, b, *sc, X, compat=True)
        assert got == ref.extend(a, b, *sc, X, compat=True), (a, b, X, sc)
        # the end is live on the last anti-diagonal, so it is never past the corner
        assert 0 <= got[1] <= len(a) and 0 <= got[2] <= len(b)
    # ALIGN composes the two compat extensions: identical reads reach both read ends
    A = "".join(rng.choice(ALPH) for _ in range(60))
    for pos in [0, 11, 40]:
        r = oracle.align(A, A, pos, pos, 17, X=5, compat=True)
        assert (r["score"], r["a_begin"], r["a_end"], r["b_begin"], r["b_end"]) == (60, 0, 60, 0, 60)
        assert r == dict(ref.align(A, A, pos, pos, 17, X=5, compat=True),
                         left=r["left"], right=r["right"])
