"""Seeded synthetic workloads for batched X-drop seed-and-extend.

This module is shared by the tests, the bench and the oracle legs.  It holds
NONE of the method's arithmetic (no scoring, no DP, no pruning): it only draws
reads, read pairs and exact shared k-mer seeds, following the recipe in
DESIGN.md §Inputs (SURVEY.md §8(d) "Generator"):

* genome: i.i.d. uniform ACGT;
* reads: uniform start, forward strand, PacBio-CLR-like errors (defaults 1.5%
  substitution, 9% insertion, 4.5% deletion per genome base: 15% total,
  indel-dominated);
* pairs: two reads whose genome intervals overlap by >= ``min_ov``;
* seed: a genome position in the overlap whose k-mer is error-free in both
  reads (tracked through genome->read maps), chosen uniformly;
* spurious pairs (fraction ``f_sp``): two reads from non-overlapping genome
  regions, with one identical k-mer planted into a copy of the second read.

Everything is a deterministic function of (config, seed).  Sequences are
returned as an ASCII uint8 pool + int64 offsets; pairs as int32[P, 4]
(a_id, b_id, a_pos, b_pos), the layout of ``xdrop_pair`` (include/xdrop.h).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

ASCII = np.frombuffer(b"ACGT", dtype=np.uint8)


@dataclasses.dataclass
class Workload:
    name: str
    seq: np.ndarray          # uint8 ASCII, all reads concatenated
    offsets: np.ndarray      # int64 [n_reads + 1]
    pairs: np.ndarray        # int32 [P, 4]  (a_id, b_id, a_pos, b_pos)
    k: int
    X: int
    M: int = 1
    mu: int = -1
    g: int = -1
    recipe: dict = dataclasses.field(default_factory=dict)

    @property
    def n_pairs(self) -> int:
        return int(self.pairs.shape[0])

    def read(self, r: int) -> bytes:
        return self.seq[self.offsets[r]:self.offsets[r + 1]].tobytes()

    def subset(self, idx) -> "Workload":
        return dataclasses.replace(self, pairs=np.ascontiguousarray(self.pairs[idx]),
                                   name=self.name + "[subset]")

    def with_X(self, X: int) -> "Workload":
        return dataclasses.replace(self, X=int(X), name=f"{self.name}@X{X}")


def _simulate_read(genome: np.ndarray, start: int, target_len: int, rng: np.random.Generator,
                   sub: float, ins: float, dele: float, k: int):
    """Simulate one read from genome[start:...].

    Returns (codes uint8, span, read_pos int64[span] (-1 if the genome base is
    not emitted as an exact copy), clean bool[span] (k-mer starting here is
    error-free and contiguous in the read)).
    """
    span = int(round(target_len / max(1e-9, 1.0 - dele + ins)))
    span = max(1, min(span, genome.shape[0] - start))
    gseg = genome[start:start + span]
    u = rng.random(span)
    is_del = u < dele
    is_sub = (u >= dele) & (u < dele + sub)
    has_ins = (rng.random(span) < ins) & ~is_del
    base = gseg.copy()
    if is_sub.any():
        base[is_sub] = (gseg[is_sub] + rng.integers(1, 4, size=int(is_sub.sum()), dtype=np.uint8)) % 4
    emit = (~is_del).astype(np.int64) + has_ins.astype(np.int64)
    pos = np.cumsum(emit) - emit                      # read position of first emitted symbol
    n = int(emit.sum())
    codes = np.empty(n, dtype=np.uint8)
    keep = ~is_del
    codes[pos[keep]] = base[keep]
    ins_idx = np.nonzero(has_ins)[0]
    codes[pos[ins_idx] + (~is_del[ins_idx]).astype(np.int64)] = rng.integers(
        0, 4, size=ins_idx.shape[0], dtype=np.uint8)
    exact = keep & ~is_sub
    read_pos = np.where(exact, pos, -1)
    # clean k-mer at p: bases p..p+k-1 exact, no insertion after p..p+k-2
    ok = exact.astype(np.int32)
    noins = (~has_ins).astype(np.int32)
    clean = np.zeros(span, dtype=bool)
    if span >= k:
        c1 = np.concatenate([[0], np.cumsum(ok)])
        c2 = np.concatenate([[0], np.cumsum(noins)])
        p = np.arange(span - k + 1)
        clean[:span - k + 1] = ((c1[p + k] - c1[p]) == k) & ((c2[p + k - 1] - c2[p]) == k - 1)
    return codes, span, read_pos, clean


def _pack_pool(reads):
    lens = np.array([r.shape[0] for r in reads], dtype=np.int64)
    off = np.zeros(len(reads) + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    seq = ASCII[np.concatenate(reads)] if reads else np.zeros(0, np.uint8)
    return np.ascontiguousarray(seq), off


def _choose_seed(rng, sa, ca, sb, cb, k):
    """Uniform genome position p in the overlap with clean k-mers in both reads."""
    lo = max(sa, sb)
    hi = min(sa + ca.shape[0], sb + cb.shape[0]) - k + 1
    if hi <= lo:
        return None
    v = ca[lo - sa:hi - sa] & cb[lo - sb:hi - sb]
    idx = np.nonzero(v)[0]
    if idx.shape[0] == 0:
        return None
    return lo + int(idx[rng.integers(0, idx.shape[0])])


def make_pool_workload(name: str, seed: int, genome_len: int, n_pairs: int, length_sampler,
                       coverage: float, min_ov: int, k: int = 17, X: int = 15,
                       sub: float = 0.015, ins: float = 0.09, dele: float = 0.045,
                       f_sp: float = 0.0, max_reads: Optional[int] = None, rc_frac: float = 0.0,
                       seeds_per_pair: int = 1) -> Workload:
    """Pool mode: reads from one genome; pairs are overlapping reads (plus spurious).
    rc_frac: fraction of reads sequenced from the reverse strand (stored reverse-
    complemented); pairs of reads from opposite strands carry XDROP_PAIR_RC.
    seeds_per_pair > 1: each overlapping pair gets that many independently drawn seeds, as
    adjacent rows (the candidate layout of xdrop_align_multiseed); n_pairs counts candidates."""
    rng = np.random.default_rng(seed)
    genome = rng.integers(0, 4, size=genome_len, dtype=np.uint8)
    mean_len = float(np.mean(length_sampler(rng, 4096)))
    n_reads = int(round(coverage * genome_len / mean_len))
    if max_reads:
        n_reads = min(n_reads, max_reads)
    lengths = length_sampler(rng, n_reads).astype(np.int64)
    starts = np.sort(rng.integers(0, max(1, genome_len - int(lengths.max())), size=n_reads))
    reads, spans, rpos, clean = [], [], [], []
    for r in range(n_reads):
        c, s, p, cl = _simulate_read(genome, int(starts[r]), int(lengths[r]), rng, sub, ins, dele, k)
        reads.append(c); spans.append(s); rpos.append(p); clean.append(cl)
    spans = np.array(spans, dtype=np.int64)
    ends = starts + spans
    # candidate overlapping pairs (i < j, starts sorted)
    cand_i, cand_j = [], []
    for i in range(n_reads):
        j_hi = np.searchsorted(starts, ends[i] - min_ov, side="left")
        js = np.arange(i + 1, j_hi)
        if js.shape[0]:
            ov = np.minimum(ends[i], ends[js]) - starts[js]
            js = js[ov >= min_ov]
            cand_i.append(np.full(js.shape[0], i)); cand_j.append(js)
    cand_i = np.concatenate(cand_i) if cand_i else np.zeros(0, np.int64)
    cand_j = np.concatenate(cand_j) if cand_j else np.zeros(0, np.int64)
    n_sp = int(round(f_sp * n_pairs))
    n_true = n_pairs - n_sp
    perm = rng.permutation(cand_i.shape[0])
    pairs = []
    for t in perm:
        if len(pairs) >= n_true * seeds_per_pair:
            break
        i, j = int(cand_i[t]), int(cand_j[t])
        if rng.random() < 0.5:
            i, j = j, i
        p = _choose_seed(rng, int(starts[i]), clean[i], int(starts[j]), clean[j], k)
        if p is None:
            continue
        pairs.append((i, j, int(rpos[i][p - starts[i]]), int(rpos[j][p - starts[j]])))
        for _ in range(seeds_per_pair - 1):
            p = _choose_seed(rng, int(starts[i]), clean[i], int(starts[j]), clean[j], k)
            pairs.append((i, j, int(rpos[i][p - starts[i]]), int(rpos[j][p - starts[j]])))
    extra = []
    tries = 0
    while len(extra) < n_sp and tries < 100 * max(1, n_sp):
        tries += 1
        i, j = int(rng.integers(0, n_reads)), int(rng.integers(0, n_reads))
        if i == j or min(ends[i], ends[j]) > max(starts[i], starts[j]):
            continue                                  # must not overlap in the genome
        li, lj = reads[i].shape[0], reads[j].shape[0]
        if li < k or lj < k:
            continue
        pa, pb = int(rng.integers(0, li - k + 1)), int(rng.integers(0, lj - k + 1))
        copy = reads[j].copy()
        copy[pb:pb + k] = reads[i][pa:pa + k]
        reads.append(copy)
        extra.append((i, len(reads) - 1, pa, pb))
    allp = pairs + extra
    if rc_frac > 0:
        # store a fraction of reads reverse-complemented and re-express every pair in stored coordinates
        flip = rng.random(len(reads)) < rc_frac
        lens = [r.shape[0] for r in reads]
        out = []
        for (i, j, pa, pb) in allp:
            fi, fj = bool(flip[i]), bool(flip[j])
            if fi and fj:                   # both reversed: an ordinary pair on the stored strand
                out.append((i, j, lens[i] - pa - k, lens[j] - pb - k))
            elif fj:                        # B reversed: revcomp(stored B) == forward B
                out.append((i, j | PAIR_RC, pa, pb))
            elif fi:                        # A reversed: swap roles, B = stored A taken reverse-complemented
                out.append((j, i | PAIR_RC, pb, pa))
            else:
                out.append((i, j, pa, pb))
        allp = out
        reads = [revcomp_codes(r) if flip[t] else r for t, r in enumerate(reads)]
    order = rng.permutation(len(allp))
    seq, off = _pack_pool(reads)
    arr = np.array(allp, dtype=np.int32).reshape(-1, 4)[order] if allp else np.zeros((0, 4), np.int32)
    recipe = dict(mode="pool", seed=seed, genome_len=genome_len, n_reads=len(reads),
                  coverage=coverage, min_ov=min_ov, k=k, X=X, sub=sub, ins=ins, dele=dele,
                  f_sp=f_sp, rc_frac=rc_frac, n_pairs=int(arr.shape[0]), mean_read_len=float(np.mean(lengths)))
    return Workload(name, seq, off, np.ascontiguousarray(arr), k, X, recipe=recipe)


def make_pair_workload(name: str, seed: int, n_pairs: int, len_lo: int, len_hi: int,
                       min_ov: int, k: int = 17, X: int = 15, sub=0.015, ins=0.09, dele=0.045,
                       f_sp: float = 0.0) -> Workload:
    """Per-pair mode: each pair has its own genome window; read 2p = A, 2p+1 = B."""
    rng = np.random.default_rng(seed)
    reads, pairs = [], []
    p = 0
    while len(pairs) < n_pairs:
        la, lb = int(rng.integers(len_lo, len_hi + 1)), int(rng.integers(len_lo, len_hi + 1))
        spurious = rng.random() < f_sp
        G = la + lb + 2 * len_hi
        genome = rng.integers(0, 4, size=G, dtype=np.uint8)
        sa = int(rng.integers(0, len_hi))
        if spurious:
            sb = sa + 2 * len_hi if sa + 2 * len_hi + lb < G else 0
        else:
            span_a = int(round(la / (1.0 - dele + ins)))
            lo_b = max(0, sa - lb + min_ov)
            hi_b = max(lo_b + 1, sa + span_a - min_ov)
            sb = int(rng.integers(lo_b, hi_b))
        ca, spa, pa_map, cla = _simulate_read(genome, sa, la, rng, sub, ins, dele, k)
        cb, spb, pb_map, clb = _simulate_read(genome, sb, lb, rng, sub, ins, dele, k)
        if spurious:
            if ca.shape[0] < k or cb.shape[0] < k:
                continue
            x, y = int(rng.integers(0, ca.shape[0] - k + 1)), int(rng.integers(0, cb.shape[0] - k + 1))
            cb = cb.copy(); cb[y:y + k] = ca[x:x + k]
            seedpair = (x, y)
        else:
            q = _choose_seed(rng, sa, cla, sb, clb, k)
            if q is None:
                continue
            seedpair = (int(pa_map[q - sa]), int(pb_map[q - sb]))
        reads += [ca, cb]
        pairs.append((2 * p, 2 * p + 1) + seedpair)
        p += 1
    seq, off = _pack_pool(reads)
    recipe = dict(mode="pairs", seed=seed, len_lo=len_lo, len_hi=len_hi, min_ov=min_ov, k=k,
                  X=X, sub=sub, ins=ins, dele=dele, f_sp=f_sp, n_pairs=n_pairs)
    return Workload(name, seq, off, np.array(pairs, dtype=np.int32), k, X, recipe=recipe)


def _normal_len(mean, sd, lo, hi):
    def f(rng, n):
        return np.clip(np.round(rng.normal(mean, sd, size=n)), lo, hi).astype(np.int64)
    return f


def _lognormal_len(median, sigma, lo, hi):
    def f(rng, n):
        return np.clip(np.round(median * np.exp(sigma * rng.standard_normal(n))), lo, hi).astype(np.int64)
    return f


def _uniform_len(lo, hi):
    def f(rng, n):
        return rng.integers(lo, hi + 1, size=n).astype(np.int64)
    return f


# ---------------------------------------------------------------- named configs
# BASELINE.json configs; SURVEY.md §8(d) table gives the concrete recipe.
def config(name: str, scale: float = 1.0, X: Optional[int] = None, seed: Optional[int] = None) -> Workload:
    """Build a named workload.  ``scale`` < 1 shrinks pair counts (tests)."""
    if name == "cfg1":      # 200 pairs, 1-2 kb, 15% error, k=17, X=15
        w = make_pair_workload("cfg1", 1 if seed is None else seed, max(1, int(200 * scale)),
                               1000, 2000, 500, k=17, X=15)
    elif name == "ecoli":   # 100k pairs of ~10 kb reads, 4.64 Mb genome, 30x
        w = make_pool_workload("ecoli", 2 if seed is None else seed, 4_641_652,
                               max(1, int(100_000 * scale)), _normal_len(10_000, 1_000, 5_000, 15_000),
                               30.0, 1_000, k=17, X=15)
    elif name == "xsweep":  # 10k pairs of 20 kb reads, f_sp = 0.2
        w = make_pool_workload("xsweep", 4 if seed is None else seed, 10_000_000,
                               max(1, int(10_000 * scale)), _normal_len(20_000, 1_000 / 3 * 3, 19_000, 21_000),
                               30.0, 5_000, k=17, X=15, f_sp=0.2)
    elif name == "celegans":  # 5M pairs, lognormal(8 kb, 0.6) in [2k, 40k], 24x of 100 Mb
        # 24x, not SURVEY's 20x: at 20x a 100 Mb genome has only ~3.6M read pairs overlapping >= 1 kb,
        # short of the 4.5M related pairs BASELINE's 5M-pair batch needs (f_sp = 0.1); 24x has ~5.2M
        w = make_pool_workload("celegans", 5 if seed is None else seed, int(100_000_000 * min(1.0, max(scale, 0.01))),
                               max(1, int(5_000_000 * scale)), _lognormal_len(8_000, 0.6, 2_000, 40_000),
                               24.0, 1_000, k=17, X=15, f_sp=0.1)
    elif name == "tiny":    # smoke: a handful of short pairs
        w = make_pair_workload("tiny", 7 if seed is None else seed, max(1, int(16 * scale)), 60, 300, 40,
                               k=17, X=15)
    else:
        raise KeyError(name)
    if X is not None:
        w = w.with_X(X)
    return w


PAIR_RC = -(1 << 31)          # bit 31 of b_id (include/xdrop.h XDROP_PAIR_RC)


def revcomp_codes(c: np.ndarray) -> np.ndarray:
    """Reverse complement of 2-bit codes A0 C1 G2 T3 (complement = 3 - code)."""
    return (3 - c[::-1]).astype(np.uint8)


def random_pairs_workload(seed: int, n_pairs: int, len_lo: int, len_hi: int, k: int, X: int,
                          M=1, mu=-1, g=-1, related=0.7, err=0.15, rc_frac=0.0) -> Workload:
    """Unstructured random pairs for parity edge cases (ragged lengths, seeds at ends).
    With rc_frac > 0 a fraction of pairs store B reverse-complemented and carry the
    XDROP_PAIR_RC flag, so that A aligns against revcomp(stored B)."""
    rng = np.random.default_rng(seed)
    reads, pairs = [], []
    for p in range(n_pairs):
        la = int(rng.integers(len_lo, len_hi + 1))
        a = rng.integers(0, 4, size=la, dtype=np.uint8)
        if rng.random() < related:
            keep = rng.random(la) >= err / 3
            b = a[keep].copy()
            subm = rng.random(b.shape[0]) < err / 3
            b[subm] = (b[subm] + rng.integers(1, 4, size=int(subm.sum()), dtype=np.uint8)) % 4
            ins_at = np.nonzero(rng.random(b.shape[0]) < err / 3)[0]
            b = np.insert(b, ins_at, rng.integers(0, 4, size=ins_at.shape[0], dtype=np.uint8))
        else:
            b = rng.integers(0, 4, size=int(rng.integers(len_lo, len_hi + 1)), dtype=np.uint8)
        if a.shape[0] < k:
            a = np.concatenate([a, rng.integers(0, 4, size=k - a.shape[0], dtype=np.uint8)])
        if b.shape[0] < k:
            b = np.concatenate([b, rng.integers(0, 4, size=k - b.shape[0], dtype=np.uint8)])
        edge = rng.random()
        if edge < 0.1:
            pa, pb = 0, 0
        elif edge < 0.2:
            pa, pb = a.shape[0] - k, b.shape[0] - k
        else:
            pa = int(rng.integers(0, a.shape[0] - k + 1))
            pb = int(rng.integers(0, b.shape[0] - k + 1))
        if rng.random() < 0.8:                       # make the seed exact
            b = b.copy(); b[pb:pb + k] = a[pa:pa + k]
        bid = 2 * p + 1
        if rc_frac and rng.random() < rc_frac:       # other strand: store revcomp(b), flag the pair
            b = revcomp_codes(b)
            bid |= PAIR_RC
        reads += [a, b]
        pairs.append((2 * p, bid, pa, pb))
    seq, off = _pack_pool(reads)
    return Workload(f"random{seed}", seq, off, np.array(pairs, dtype=np.int32).reshape(-1, 4), k, X, M, mu, g,
                    recipe=dict(mode="random", seed=seed, len_lo=len_lo, len_hi=len_hi, related=related))
