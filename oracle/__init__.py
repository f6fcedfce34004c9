"""CPU oracle for batched X-drop seed-and-extend (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2309_07270_b200`` never imports it, and it never imports the product.

Two independent implementations of the same written reading (DESIGN.md
"Readings"; paper anchors PAPER.md:73-74, 81, 85-89, 224, 327):

* ``xdrop_oracle.c`` -- plain C, built to ``liboracle.so``; loaded here with
  ctypes (``extend``, ``align``, ``align_batch``).
* ``xdrop_ref.py``   -- pure-Python twin (dict-based) plus FULLDP, used for
  tiny brute-force pins.

Pins (tests/test_oracle_pins.py): brute-force enumeration of all alignments on
tiny inputs, FULLDP equality once X exceeds the bound, closed forms (identical
strings, single substitution, all-mismatch cell count), hand-traced golden
fixtures under tests/golden/, upper bound, symmetry, achievability.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xdrop_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class Ext(ctypes.Structure):
    _fields_ = [("best", ctypes.c_int32), ("istar", ctypes.c_int32),
                ("jstar", ctypes.c_int32), ("cells", ctypes.c_int64)]


class Result(ctypes.Structure):
    _fields_ = [("score", ctypes.c_int32), ("a_begin", ctypes.c_int32),
                ("a_end", ctypes.c_int32), ("b_begin", ctypes.c_int32),
                ("b_end", ctypes.c_int32)]


RESULT_DTYPE = np.dtype([("score", "<i4"), ("a_begin", "<i4"), ("a_end", "<i4"),
                         ("b_begin", "<i4"), ("b_end", "<i4")])


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_extend.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p,
                                          ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.POINTER(Ext)]
            lib.oracle_align.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.POINTER(Result),
                                         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(Ext),
                                         ctypes.POINTER(Ext)]
            lib.oracle_align_batch.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int64] + \
                [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int64)]
            lib.oracle_extend_mode.argtypes = lib.oracle_extend.argtypes[:8] + \
                [ctypes.c_int, ctypes.POINTER(Ext)]
            lib.oracle_align_mode.argtypes = lib.oracle_align.argtypes[:11] + [ctypes.c_int] + \
                lib.oracle_align.argtypes[11:]
            lib.oracle_align_batch_mode.argtypes = lib.oracle_align_batch.argtypes[:12] + \
                [ctypes.c_int] + lib.oracle_align_batch.argtypes[12:]
            _lib = lib
    return _lib


def _b(s) -> bytes:
    return s.encode() if isinstance(s, str) else bytes(s)


def extend(a, b, M=1, mu=-1, g=-1, X=15, compat=False):
    """EXTEND(a, b) -> (best, i*, j*, cells)   (C oracle).  compat=True: the SeqAn/LOGAN-style
    mode (Q28-Q30) -> (H of the longest extension, its i, j, cells)."""
    a, b = _b(a), _b(b)
    out = Ext()
    rc = _load().oracle_extend_mode(a, len(a), b, len(b), M, mu, g, X, int(compat), ctypes.byref(out))
    if rc:
        raise RuntimeError(f"oracle_extend failed: {rc}")
    return out.best, out.istar, out.jstar, out.cells


def align(A, B, a_pos, b_pos, k, M=1, mu=-1, g=-1, X=15, compat=False):
    """ALIGN one pair -> dict(score, a_begin, a_end, b_begin, b_end, cells, left, right)."""
    A, B = _b(A), _b(B)
    r, c, L, R = Result(), ctypes.c_int64(), Ext(), Ext()
    rc = _load().oracle_align_mode(A, len(A), B, len(B), a_pos, b_pos, k, M, mu, g, X, int(compat),
                                   ctypes.byref(r), ctypes.byref(c), ctypes.byref(L),
                                   ctypes.byref(R))
    if rc:
        raise ValueError(f"oracle_align failed: {rc}")
    return dict(score=r.score, a_begin=r.a_begin, a_end=r.a_end, b_begin=r.b_begin,
                b_end=r.b_end, cells=c.value, left=(L.best, L.istar, L.jstar, L.cells),
                right=(R.best, R.istar, R.jstar, R.cells))


def align_batch(seqA: np.ndarray, offA: np.ndarray, seqB: np.ndarray, offB: np.ndarray,
                pairs: np.ndarray, k: int, M=1, mu=-1, g=-1, X=15, nthreads=None,
                order: np.ndarray | None = None, compat=False):
    """Batch ALIGN over read pools (uint8 ASCII + int64 offsets, pairs int32[n,4]).
    compat=True: the SeqAn/LOGAN-style mode (Q28-Q30).

    Returns (results structured array RESULT_DTYPE[n], cells int64[n]).
    """
    seqA = np.ascontiguousarray(seqA, dtype=np.uint8)
    seqB = np.ascontiguousarray(seqB, dtype=np.uint8)
    offA = np.ascontiguousarray(offA, dtype=np.int64)
    offB = np.ascontiguousarray(offB, dtype=np.int64)
    pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 4)
    n = pairs.shape[0]
    out = np.zeros(n, dtype=RESULT_DTYPE)
    cells = np.zeros(n, dtype=np.int64)
    if order is not None:
        order = np.ascontiguousarray(order, dtype=np.int64)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    err = ctypes.c_int64(-1)
    rc = _load().oracle_align_batch_mode(
        seqA.ctypes.data, offA.ctypes.data, seqB.ctypes.data, offB.ctypes.data,
        pairs.ctypes.data, order.ctypes.data if order is not None else None, n,
        k, M, mu, g, X, int(compat), out.ctypes.data, cells.ctypes.data, int(nthreads), ctypes.byref(err))
    if rc:
        raise ValueError(f"oracle_align_batch failed rc={rc} at pair {err.value}")
    return out, cells


def best_seed(pairs: np.ndarray, scores: np.ndarray) -> np.ndarray:
    """Several seeds per candidate pair (reading Q26): a candidate
    is a maximal run of adjacent rows with equal (a_id, b_id) (strand bit included); every row
    gets the index of its candidate's highest-scoring row, ties to the first.  Plain loop."""
    pairs = np.asarray(pairs).reshape(-1, 4)
    n = pairs.shape[0]
    best = np.zeros(n, dtype=np.int64)
    i = 0
    while i < n:
        j = i
        while j + 1 < n and pairs[j + 1, 0] == pairs[i, 0] and pairs[j + 1, 1] == pairs[i, 1]:
            j += 1
        b = i
        for t in range(i + 1, j + 1):
            if scores[t] > scores[b]:
                b = t
        best[i:j + 1] = b
        i = j + 1
    return best
