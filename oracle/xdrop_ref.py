"""Pure-Python twin of the X-drop oracle, plus FULLDP (TEST INFRASTRUCTURE ONLY).

Same written reading as ``xdrop_oracle.c`` (SURVEY.md
§8(c)), written a second time in a
different style (dicts keyed by (i, j), Python sets for the live sets L_d) so
the two oracle implementations share no code.  Small inputs only.
"""
from __future__ import annotations


def s(x: str, y: str, M: int, mu: int) -> int:
    """Substitution score: M on a (case-insensitive) match, mu otherwise (reading Q10)."""
    return M if x.upper() == y.upper() else mu


def extend(a: str, b: str, M=1, mu=-1, g=-1, X=15, compat=False):
    """EXTEND(a, b) -> (best, i*, j*, cells); anti-diagonal X-drop (reading Q1-Q8).

    compat=True: the SeqAn/LOGAN-style mode (Q28-Q30): a pure-gap
    cell (i = 0 or j = 0) lives only if v > best - X; the result is the "longest extension", the
    largest-H live cell of the last anti-diagonal that has one (smallest i on ties), with its H."""
    m, n = len(a), len(b)
    H = {(0, 0): 0}
    live = {0: {0}, -1: set()}          # L_d as sets of i
    best, istar, jstar, cells = 0, 0, 0, 1
    last = (0, 0, 0)                    # compat: (H, i, j) of the last live anti-diagonal's max
    for d in range(1, m + n + 1):
        L1, L2 = live[d - 1], live[d - 2]
        if not L1 and not L2:
            break
        los = [min(L1)] if L1 else []
        his = [max(L1) + 1] if L1 else []
        if L2:
            los.append(min(L2) + 1)
            his.append(max(L2) + 1)
        lo = max(0, d - n, min(los))
        hi = min(m, d, max(his))
        cells += max(0, hi - lo + 1)
        thr = best - X                   # best over anti-diagonals < d (reading Q2)
        Ld = set()
        for i in range(lo, hi + 1):
            j = d - i
            cand = []
            if i - 1 in L1:
                cand.append(H[(i - 1, j)] + g)
            if i in L1 and j >= 1:
                cand.append(H[(i, j - 1)] + g)
            if i - 1 in L2 and j >= 1:
                cand.append(H[(i - 1, j - 1)] + s(a[i - 1], b[j - 1], M, mu))
            if cand:
                v = max(cand)
                on_edge = i == 0 or j == 0
                if (v > thr) if (compat and on_edge) else (v >= thr):   # Q3; Q28 (compat edge)
                    H[(i, j)] = v
                    Ld.add(i)
        live[d] = Ld
        if Ld:
            vstar = max(H[(i, d - i)] for i in Ld)
            iv = min(i for i in Ld if H[(i, d - i)] == vstar)
            if vstar > best:             # reading Q8: strict, then smallest i
                best, istar, jstar = vstar, iv, d - iv
            last = (vstar, iv, d - iv)   # Q29
    if compat:
        return last + (cells,)           # Q29, Q30: the longest extension and its H
    return best, istar, jstar, cells


def fulldp(a: str, b: str, M=1, mu=-1, g=-1):
    """FULLDP: the same recurrence over the whole rectangle, no pruning.

    Returns (max H, i*, j*) with ties broken by smallest anti-diagonal, then
    smallest i (SURVEY.md §8(c) FULLDP).  Plain Needleman-Wunsch table.
    """
    m, n = len(a), len(b)
    H = [[0] * (n + 1) for _ in range(m + 1)]
    for i in range(1, m + 1):
        H[i][0] = H[i - 1][0] + g
    for j in range(1, n + 1):
        H[0][j] = H[0][j - 1] + g
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            H[i][j] = max(H[i - 1][j] + g, H[i][j - 1] + g,
                          H[i - 1][j - 1] + s(a[i - 1], b[j - 1], M, mu))
    best = None
    for d in range(0, m + n + 1):
        for i in range(max(0, d - n), min(m, d) + 1):
            v = H[i][d - i]
            if best is None or v > best[0]:
                best = (v, i, d - i)
    return best


def revcomp(B: str) -> str:
    """Reverse complement (reading Q16: a pair may use B on the other strand)."""
    comp = {"A": "T", "C": "G", "G": "C", "T": "A"}
    return "".join(comp[c.upper()] for c in reversed(B))


def align(A: str, B: str, a_pos: int, b_pos: int, k: int, M=1, mu=-1, g=-1, X=15, rc=False,
          compat=False):
    """ALIGN (reading Q9, Q13): seed columns + right EXTEND + left EXTEND on reversals.
    rc=True aligns A against revcomp(B); b_pos / b_begin / b_end are revcomp(B) coordinates.
    compat=True: both extensions in the SeqAn/LOGAN-style mode (Q28-Q30)."""
    if rc:
        B = revcomp(B)
    seed = sum(s(A[a_pos + t], B[b_pos + t], M, mu) for t in range(k))
    R = extend(A[a_pos + k:], B[b_pos + k:], M, mu, g, X, compat)
    L = extend(A[:a_pos][::-1], B[:b_pos][::-1], M, mu, g, X, compat)
    return dict(score=L[0] + seed + R[0], a_begin=a_pos - L[1], b_begin=b_pos - L[2],
                a_end=a_pos + k + R[1], b_end=b_pos + k + R[2], cells=L[3] + R[3])
