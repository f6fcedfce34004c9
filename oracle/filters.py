"""CPU oracle of the candidate-pair filters (TEST INFRASTRUCTURE ONLY; same rules as oracle/__init__.py:
only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import it).  Plain Python, no code
shared with the CUDA path (paper_2309_07270_b200/csrc/xdrop_filters.cu).

* adaptive_keep  -- f2, BELLA's adaptive X-drop threshold ("An adaptive threshold is used to perform
  the X-drop alignment", §II).  The paper gives no formula: DESIGN.md reading Q12.
  ov = min(a_pos, b_pos) + min(|A| - a_pos, |B| - b_pos), mu = phi * ov,
  keep iff score >= mu - sqrt(c * mu), in IEEE double precision (Python floats), in that order.
* seed_kmer_freq -- f4, the k-mer frequency band of ELBA's seeds (LOWER_KMER_FREQ=20,
  UPPER_KMER_FREQ=30/50, §IV-A).  The count of a seed k-mer is the number of positions
  of the pool's reads whose k-mer equals it on either strand (canonical k-mer = the lexicographically
  smaller of the k-mer and its reverse complement over A < C < G < T; k-mers with a non-ACGT base or
  crossing a read boundary are not counted).  keep iff lower <= count <= upper.
"""
from __future__ import annotations

import math

import numpy as np

_COMP = {"A": "T", "C": "G", "G": "C", "T": "A"}


def overlap_estimate(offA, offB, pair) -> int:
    """Bases of the overlap the seed's diagonal implies (reading Q12)."""
    a_id, b_id, a_pos, b_pos = (int(x) for x in pair)
    b_id &= 0x7fffffff
    la = int(offA[a_id + 1] - offA[a_id])
    lb = int(offB[b_id + 1] - offB[b_id])
    return min(a_pos, b_pos) + min(la - a_pos, lb - b_pos)


def adaptive_keep(offA, offB, pairs, scores, phi: float, c: float) -> np.ndarray:
    """f2: keep[p] = score[p] >= phi*ov - sqrt(c * phi*ov)   (plain loop, double precision)."""
    pairs = np.asarray(pairs).reshape(-1, 4)
    keep = np.zeros(pairs.shape[0], dtype=np.uint8)
    for p in range(pairs.shape[0]):
        ov = overlap_estimate(offA, offB, pairs[p])
        mu = float(phi) * float(ov)
        t = mu - math.sqrt(float(c) * mu)
        keep[p] = 1 if float(scores[p]) >= t else 0
    return keep


def canonical(kmer: str) -> str | None:
    """The canonical form of a k-mer, or None if it holds a base outside ACGT (either case)."""
    kmer = kmer.upper()
    if any(ch not in _COMP for ch in kmer):
        return None
    rc = "".join(_COMP[ch] for ch in reversed(kmer))
    return min(kmer, rc)


def kmer_counts(seq, offsets, k: int) -> dict:
    """Counts of every canonical k-mer over all positions of all reads (plain dict; small pools)."""
    text = bytes(np.asarray(seq, dtype=np.uint8)).decode("ascii")
    counts: dict = {}
    for r in range(len(offsets) - 1):
        read = text[int(offsets[r]):int(offsets[r + 1])]
        for x in range(len(read) - k + 1):
            cf = canonical(read[x:x + k])
            if cf is not None:
                counts[cf] = counts.get(cf, 0) + 1
    return counts


def seed_kmer_freq(seq, offsets, pairs, k: int, lower: int, upper: int):
    """f4: (freq int32[n], keep uint8[n]) of each pair's seed k-mer A[a_pos, a_pos + k)."""
    pairs = np.asarray(pairs).reshape(-1, 4)
    counts = kmer_counts(seq, offsets, k)
    text = bytes(np.asarray(seq, dtype=np.uint8)).decode("ascii")
    freq = np.zeros(pairs.shape[0], dtype=np.int32)
    for p in range(pairs.shape[0]):
        a_id, a_pos = int(pairs[p, 0]), int(pairs[p, 2])
        x = int(offsets[a_id]) + a_pos
        cf = canonical(text[x:x + k])
        if cf is None:
            raise ValueError(f"pair {p}: seed holds a base outside ACGT")
        freq[p] = counts.get(cf, 0)
    keep = ((freq >= lower) & (freq <= upper)).astype(np.uint8)
    return freq, keep
