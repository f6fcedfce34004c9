"""ctypes binding of libxdrop.so (include/xdrop.h).  Argument marshalling only.

Every compute step runs inside the CUDA library; there is no Python or CPU
fallback.  If the shared library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XDROP_LIB") or os.path.join(HERE, "libxdrop.so")   # XDROP_LIB: A/B experiments

# status codes (xdrop_status)
OK, EINVAL, ENOMEM, ECUDA, EALPHABET, ESEED, ELENGTH, ESTATE, ENODEV = 0, -1, -2, -3, -4, -5, -6, -7, -8
POLICIES = {"cells": 0, "one2all": 1, "one2one": 2, "opt_one2one": 3, "mixed": 3}
FLAG_FORCE_WIDE, FLAG_FORCE_GENERAL, FLAG_NO_SORT, FLAG_TIERED, FLAG_SHARED = 1, 2, 4, 8, 16
FLAG_SEQAN_COMPAT = 32     # SeqAn/LOGAN-style conventions (include/xdrop.h; Q28-Q30)
KERNELS = {"auto": 0, "tiered": FLAG_TIERED, "shared": FLAG_SHARED}   # packed band kernel (include/xdrop.h)
MAX_READ_LEN = 1 << 18

RESULT_DTYPE = np.dtype([("score", "<i4"), ("a_begin", "<i4"), ("a_end", "<i4"),
                         ("b_begin", "<i4"), ("b_end", "<i4")])


class Params(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32), ("gap", ctypes.c_int32),
                ("xdrop", ctypes.c_int32), ("k", ctypes.c_int32)]


class InitOpts(ctypes.Structure):
    _fields_ = [("devices", ctypes.POINTER(ctypes.c_int)), ("n_devices", ctypes.c_int),
                ("policy", ctypes.c_int), ("n_ranks", ctypes.c_int), ("batch_size", ctypes.c_int),
                ("subbatches", ctypes.c_int), ("flags", ctypes.c_int)]


class Seqs(ctypes.Structure):
    _fields_ = [("seq", ctypes.c_void_p), ("offsets", ctypes.c_void_p), ("n", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("items", ctypes.c_int64), ("escalated", ctypes.c_int64 * 4), ("cells", ctypes.c_int64),
                ("kernel_ms", ctypes.c_float), ("total_ms", ctypes.c_float), ("pack_ms", ctypes.c_float),
                ("launches", ctypes.c_int64), ("level_ms", ctypes.c_float * 4),
                ("level_cells", ctypes.c_int64 * 4), ("level_items", ctypes.c_int64 * 4),
                ("long_items", ctypes.c_int64), ("stolen", ctypes.c_int64), ("band_kernel", ctypes.c_int64), ("cta_items", ctypes.c_int64), ("cta4k_items", ctypes.c_int64), ("endgame_stolen", ctypes.c_int64),
                ("probe_overflows", ctypes.c_int64)]


class TraceEvent(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("gpu", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("sub", ctypes.c_int32), ("n_pairs", ctypes.c_int64), ("t0_ms", ctypes.c_double),
                ("t1_ms", ctypes.c_double)]


class SchedStats(ctypes.Structure):
    _fields_ = [("handoffs", ctypes.c_int64), ("exchange_msgs", ctypes.c_int64), ("turns", ctypes.c_int64),
                ("span_ms", ctypes.c_double), ("busy_ms", ctypes.c_double * 16),
                ("max_concurrent", ctypes.c_int32), ("n_events", ctypes.c_int32)]


TRACE_DTYPE = np.dtype([("rank", "<i4"), ("gpu", "<i4"), ("batch", "<i4"), ("sub", "<i4"),
                        ("n_pairs", "<i8"), ("t0_ms", "<f8"), ("t1_ms", "<f8")])

EXPORTS = [
    "xdrop_init", "xdrop_align_batch", "xdrop_align_batch_device", "xdrop_last_stats",
    "xdrop_best_seed_device", "xdrop_align_multiseed",
    "xdrop_last_sched_stats", "xdrop_last_trace", "xdrop_sched_simulate", "xdrop_ring_left",
    "xdrop_ring_right", "xdrop_finalize", "xdrop_strerror", "xdrop_last_error_index", "xdrop_alu_peaks",
    "xdrop_last_timeline", "xdrop_pool_register", "xdrop_align_pooled", "xdrop_pool_release",
    "xdrop_adaptive_filter_device", "xdrop_seed_kmer_freq_device", "xdrop_ring_turn_next", "xdrop_ring_turn_prev",
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(no CPU fallback exists by design)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.xdrop_init.argtypes = [ctypes.POINTER(InitOpts), ctypes.POINTER(P)]
    lib.xdrop_align_batch.argtypes = [P, ctypes.POINTER(Seqs), ctypes.POINTER(Seqs), P, ctypes.c_int64,
                                      ctypes.POINTER(Params), P, P]
    lib.xdrop_align_batch_device.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int64, P, P, ctypes.c_int64,
                                             ctypes.c_int64, P, ctypes.c_int64, ctypes.POINTER(Params), P, P, P]
    lib.xdrop_last_stats.argtypes = [P, ctypes.POINTER(Stats)]
    lib.xdrop_best_seed_device.argtypes = [P, P, P, ctypes.c_int64, P, P]
    lib.xdrop_align_multiseed.argtypes = [P, ctypes.POINTER(Seqs), ctypes.POINTER(Seqs), P, ctypes.c_int64,
                                          ctypes.POINTER(Params), P, P, P]
    lib.xdrop_last_sched_stats.argtypes = [P, ctypes.POINTER(SchedStats)]
    lib.xdrop_last_trace.argtypes = [P, P, ctypes.c_int64]
    lib.xdrop_last_trace.restype = ctypes.c_int64
    lib.xdrop_sched_simulate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         P, ctypes.c_int64, ctypes.c_double, ctypes.POINTER(SchedStats), P,
                                         ctypes.c_int64, P]
    lib.xdrop_sched_simulate.restype = ctypes.c_int64
    lib.xdrop_ring_left.argtypes = [ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
    lib.xdrop_ring_right.argtypes = [ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
    lib.xdrop_ring_turn_next.argtypes = [ctypes.c_int] * 3 + [P, ctypes.c_int, ctypes.c_int, P, P]
    lib.xdrop_ring_turn_prev.argtypes = [ctypes.c_int] * 3 + [P, ctypes.c_int, ctypes.c_int]
    lib.xdrop_finalize.argtypes = [P]
    lib.xdrop_strerror.argtypes = [ctypes.c_int]
    lib.xdrop_strerror.restype = ctypes.c_char_p
    lib.xdrop_last_error_index.argtypes = [P]
    lib.xdrop_last_error_index.restype = ctypes.c_int64
    lib.xdrop_alu_peaks.argtypes = [ctypes.c_int, P, ctypes.c_int]
    lib.xdrop_pool_register.argtypes = [P, ctypes.POINTER(Seqs), ctypes.POINTER(ctypes.c_int32)]
    lib.xdrop_align_pooled.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int64,
                                       ctypes.POINTER(Params), P, P]
    lib.xdrop_pool_release.argtypes = [P, ctypes.c_int32]
    lib.xdrop_adaptive_filter_device.argtypes = [P, ctypes.c_int64, P, ctypes.c_int64, P, P, ctypes.c_int64,
                                                 ctypes.c_double, ctypes.c_double, P, P, P]
    lib.xdrop_seed_kmer_freq_device.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int64,
                                                ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P]
    lib.xdrop_last_timeline.argtypes = [P, P, ctypes.c_int64]
    lib.xdrop_last_timeline.restype = ctypes.c_int64
    return lib


lib = _load()


class XdropError(RuntimeError):
    def __init__(self, status: int, where: str, index: int = -1):
        self.status, self.index = status, index
        msg = lib.xdrop_strerror(status).decode()
        super().__init__(f"{where}: {msg} (status {status}, index {index})")


def check(status: int, where: str, ctx=None):
    if status != OK:
        idx = lib.xdrop_last_error_index(ctx) if ctx else -1
        raise XdropError(status, where, idx)
