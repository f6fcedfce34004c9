"""B200-native batched X-drop seed-and-extend (arxiv 2309.07270's hot path).

Public API: :class:`Aligner` (wraps the C ABI in include/xdrop.h).  PyTorch is
used only for device memory and streams (``align_device``); every step of the
path runs in the CUDA kernels of ``libxdrop.so``.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from ._native import RESULT_DTYPE, TRACE_DTYPE, XdropError  # noqa: F401

__all__ = ["Aligner", "Pipeline", "XdropError", "RESULT_DTYPE", "TRACE_DTYPE", "ring_left", "ring_right",
           "sched_simulate", "alu_peaks", "pair_costs", "shard_pairs", "adaptive_filter_device",
           "seed_kmer_freq_device"]


def _params(M, mu, g, X, k):
    return N.Params(int(M), int(mu), int(g), int(X), int(k))


class Aligner:
    """A context over one or more GPUs (``xdrop_init``)."""

    def __init__(self, n_devices: int = 1, devices=None, policy: str = "cells", n_ranks: int = 1,
                 batch_size: int = 10000, subbatches: int = 1, flags: int = 0, kernel: str = "auto",
                 seqan_compat: bool = False):
        """kernel: packed band kernel -- "auto" (per batch, from the on-device probe's escalation estimate),
        "tiered" or "shared" (XDROP_FLAG_TIERED / XDROP_FLAG_SHARED).
        seqan_compat: SeqAn/LOGAN-style conventions (XDROP_FLAG_SEQAN_COMPAT; Q28-Q30)."""
        flags |= N.KERNELS[kernel]
        if seqan_compat:
            flags |= N.FLAG_SEQAN_COMPAT
        opts = N.InitOpts()
        self._dev_arr = None
        if devices is not None:
            self._dev_arr = (ctypes.c_int * len(devices))(*devices)
            opts.devices = ctypes.cast(self._dev_arr, ctypes.POINTER(ctypes.c_int))
            n_devices = len(devices)
        opts.n_devices = n_devices
        opts.policy = N.POLICIES[policy] if isinstance(policy, str) else int(policy)
        opts.n_ranks, opts.batch_size, opts.subbatches, opts.flags = n_ranks, batch_size, subbatches, flags
        h = ctypes.c_void_p()
        N.check(N.lib.xdrop_init(ctypes.byref(opts), ctypes.byref(h)), "xdrop_init")
        self._h = h
        self._device0 = int(devices[0]) if devices is not None else 0   # device of align_device

    def close(self):
        if getattr(self, "_h", None):
            N.lib.xdrop_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---------------------------------------------------------------- host API
    def align(self, seqA: np.ndarray, offA: np.ndarray, pairs: np.ndarray, k: int, X: int,
              M: int = 1, mu: int = -1, g: int = -1, seqB=None, offB=None, want_cells: bool = True):
        """xdrop_align_batch on host buffers -> (results RESULT_DTYPE[n], cells int64[n])."""
        seqA = np.ascontiguousarray(seqA, dtype=np.uint8)
        offA = np.ascontiguousarray(offA, dtype=np.int64)
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 4)
        A = N.Seqs(seqA.ctypes.data, offA.ctypes.data, offA.shape[0] - 1)
        if seqB is None:
            B = A
            pB = ctypes.byref(A)
        else:
            seqB = np.ascontiguousarray(seqB, dtype=np.uint8)
            offB = np.ascontiguousarray(offB, dtype=np.int64)
            B = N.Seqs(seqB.ctypes.data, offB.ctypes.data, offB.shape[0] - 1)
            pB = ctypes.byref(B)
        n = pairs.shape[0]
        # every element is written by the call (on error the buffers are unspecified: include/xdrop.h)
        out = np.empty(n, dtype=RESULT_DTYPE)
        cells = np.empty(n, dtype=np.int64) if want_cells else None
        p = _params(M, mu, g, X, k)
        st = N.lib.xdrop_align_batch(self._h, ctypes.byref(A), pB, pairs.ctypes.data, n, ctypes.byref(p),
                                     out.ctypes.data, cells.ctypes.data if want_cells else None)
        N.check(st, "xdrop_align_batch", self._h)
        return out, cells

    # ------------------------------------------------------ registered pools
    def register_pool(self, seq: np.ndarray, offsets: np.ndarray) -> int:
        """xdrop_pool_register: upload + 2-bit pack a host read pool once (every device of the
        context); returns the pool id for align_pooled."""
        seq = np.ascontiguousarray(seq, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        S = N.Seqs(seq.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1)
        pid = ctypes.c_int32(-1)
        N.check(N.lib.xdrop_pool_register(self._h, ctypes.byref(S), ctypes.byref(pid)), "xdrop_pool_register",
                self._h)
        return int(pid.value)

    def release_pool(self, pool_id: int):
        N.check(N.lib.xdrop_pool_release(self._h, int(pool_id)), "xdrop_pool_release")

    def align_pooled(self, pool_id: int, pairs: np.ndarray, k: int, X: int, M: int = 1, mu: int = -1, g: int = -1,
                     pool_b: int | None = None, want_cells: bool = True):
        """xdrop_align_pooled on registered pools -> (results RESULT_DTYPE[n], cells int64[n])."""
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 4)
        n = pairs.shape[0]
        out = np.empty(n, dtype=RESULT_DTYPE)
        cells = np.empty(n, dtype=np.int64) if want_cells else None
        p = _params(M, mu, g, X, k)
        st = N.lib.xdrop_align_pooled(self._h, int(pool_id), int(pool_id if pool_b is None else pool_b),
                                      pairs.ctypes.data, n, ctypes.byref(p), out.ctypes.data,
                                      cells.ctypes.data if want_cells else None)
        N.check(st, "xdrop_align_pooled", self._h)
        return out, cells

    # -------------------------------------------------------------- device API
    def align_device(self, seqA, offA, pairs, out, cells, k: int, X: int, M: int = 1, mu: int = -1,
                     g: int = -1, seqB=None, offB=None, lenA: int | None = None, lenB: int | None = None,
                     stream=None):
        """xdrop_align_batch_device on torch CUDA tensors (uint8 pool, int64 offsets,
        int32[n,4] pairs, int32[n,5] out, int64[n] cells or None)."""
        if seqB is None:
            seqB, offB = seqA, offA
        n = int(pairs.shape[0]) if pairs.dim() == 2 else -1
        _check_tensor("seqA", seqA, (1,), ("uint8", "int8"), self._device0)
        _check_tensor("offA", offA, (1,), ("int64",), self._device0)
        _check_tensor("seqB", seqB, (1,), ("uint8", "int8"), self._device0)
        _check_tensor("offB", offB, (1,), ("int64",), self._device0)
        _check_tensor("pairs", pairs, (2,), ("int32",), self._device0, cols=4)
        _check_tensor("out", out, (2,), ("int32",), self._device0, rows=n, cols=5)
        if cells is not None:
            _check_tensor("cells", cells, (1,), ("int64",), self._device0, rows=n)
        if offA.shape[0] < 1 or offB.shape[0] < 1:
            raise ValueError("offsets need n+1 >= 1 entries")
        nA = offA.shape[0] - 1
        if lenA is None:
            lenA = int(seqA.shape[0])
        if seqB is seqA and offB is offA:
            nB, lenB = nA, lenA
        else:
            nB = offB.shape[0] - 1
            lenB = int(seqB.shape[0]) if lenB is None else lenB
        if not (0 <= lenA <= seqA.shape[0] and 0 <= lenB <= seqB.shape[0]):
            raise ValueError("lenA / lenB exceed the pool tensors")
        p = _params(M, mu, g, X, k)
        s = stream.cuda_stream if stream is not None else None
        st = N.lib.xdrop_align_batch_device(
            self._h, seqA.data_ptr(), offA.data_ptr(), nA, lenA, seqB.data_ptr(), offB.data_ptr(), nB, lenB,
            pairs.data_ptr(), pairs.shape[0], ctypes.byref(p), out.data_ptr(),
            cells.data_ptr() if cells is not None else None, s)
        N.check(st, "xdrop_align_batch_device", self._h)

    # ------------------------------------------------- several seeds per pair (f4)
    def align_multiseed(self, seqA: np.ndarray, offA: np.ndarray, pairs: np.ndarray, k: int, X: int,
                        M: int = 1, mu: int = -1, g: int = -1, seqB=None, offB=None):
        """xdrop_align_multiseed: every row aligned as by align(), plus best int64[n] = the row of
        each row's candidate (adjacent rows with equal a_id, b_id) with the highest score."""
        seqA = np.ascontiguousarray(seqA, dtype=np.uint8)
        offA = np.ascontiguousarray(offA, dtype=np.int64)
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 4)
        A = N.Seqs(seqA.ctypes.data, offA.ctypes.data, offA.shape[0] - 1)
        if seqB is None:
            pB = ctypes.byref(A)
        else:
            seqB = np.ascontiguousarray(seqB, dtype=np.uint8)
            offB = np.ascontiguousarray(offB, dtype=np.int64)
            B = N.Seqs(seqB.ctypes.data, offB.ctypes.data, offB.shape[0] - 1)
            pB = ctypes.byref(B)
        n = pairs.shape[0]
        out = np.zeros(n, dtype=RESULT_DTYPE)
        cells = np.zeros(n, dtype=np.int64)
        best = np.zeros(n, dtype=np.int64)
        p = _params(M, mu, g, X, k)
        st = N.lib.xdrop_align_multiseed(self._h, ctypes.byref(A), pB, pairs.ctypes.data, n, ctypes.byref(p),
                                         out.ctypes.data, best.ctypes.data, cells.ctypes.data)
        N.check(st, "xdrop_align_multiseed", self._h)
        return out, best, cells

    def best_seed_device(self, pairs, out, best, stream=None):
        """xdrop_best_seed_device on torch CUDA tensors: pairs int32[n,4], out int32[n,5] (as
        written by align_device), best int64[n]."""
        s = stream.cuda_stream if stream is not None else None
        st = N.lib.xdrop_best_seed_device(self._h, pairs.data_ptr(), out.data_ptr(), pairs.shape[0],
                                          best.data_ptr(), s)
        N.check(st, "xdrop_best_seed_device", self._h)

    # ------------------------------------------------------------ observability
    def stats(self) -> dict:
        s = N.Stats()
        N.check(N.lib.xdrop_last_stats(self._h, ctypes.byref(s)), "xdrop_last_stats")
        return dict(items=s.items, escalated=list(s.escalated), kernel_ms=s.kernel_ms, total_ms=s.total_ms,
                    pack_ms=s.pack_ms, launches=s.launches, level_ms=list(s.level_ms),
                    level_cells=list(s.level_cells), level_items=list(s.level_items),
                    long_items=s.long_items, stolen=s.stolen, cells=s.cells,
                    band_kernel=("merged32", "tiered", "shared")[s.band_kernel], cta_items=s.cta_items, cta4k_items=s.cta4k_items, endgame_stolen=s.endgame_stolen,
                    probe_overflows=s.probe_overflows)

    def sched_stats(self) -> dict:
        s = N.SchedStats()
        N.check(N.lib.xdrop_last_sched_stats(self._h, ctypes.byref(s)), "xdrop_last_sched_stats")
        return dict(handoffs=s.handoffs, exchange_msgs=s.exchange_msgs, turns=s.turns, span_ms=s.span_ms,
                    busy_ms=list(s.busy_ms), max_concurrent=s.max_concurrent)

    def trace(self) -> np.ndarray:
        n = N.lib.xdrop_last_trace(self._h, None, 0)
        buf = np.zeros(max(n, 0), dtype=TRACE_DTYPE)
        if n > 0:
            N.lib.xdrop_last_trace(self._h, buf.ctypes.data, n)
        return buf

    def timeline(self) -> np.ndarray:
        """Work units of the last call's band kernel (XDROP_TIMELINE=1 at construction):
        rows (type, warp, start_ns, end_ns)."""
        n = N.lib.xdrop_last_timeline(self._h, None, 0)
        buf = np.zeros((max(n, 0), 3), dtype=np.uint64)
        if n > 0:
            N.lib.xdrop_last_timeline(self._h, buf.ctypes.data, n)
        out = np.zeros((buf.shape[0], 4), dtype=np.int64)
        out[:, 0] = (buf[:, 0] & 0xFF).astype(np.int64)
        out[:, 1] = (buf[:, 0] >> 8).astype(np.int64)
        out[:, 2:] = buf[:, 1:].astype(np.int64)
        return out



PEAK_PROBES = ("VIMNMX3.S16x2", "VIMNMX3", "LOP3", "IADD3", "IMAD", "VIMNMX3.S16x2+IMAD")


class Pipeline:
    """Several host-API batches in flight on one GPU (a serving loop): ``n_inflight`` independent
    contexts (``xdrop_init`` each: own device workspaces and stream), each driven by its own host
    thread, so one batch's host-to-device upload and pack overlap another's band kernels and the
    next batch's kernels fill the SMs a batch's tail leaves idle.  Every batch is one complete
    ``Aligner.align`` call (its H2D, kernels and D2H); results are the same as the serial calls'.
    ctypes releases the GIL for the duration of each C call.  DESIGN.md §9."""

    def __init__(self, n_inflight: int = 3, **aligner_kwargs):
        import queue
        from concurrent.futures import ThreadPoolExecutor
        self._free = queue.Queue()
        self._als = [Aligner(**aligner_kwargs) for _ in range(max(1, int(n_inflight)))]
        for al in self._als:
            self._free.put(al)
        self._pool = ThreadPoolExecutor(max_workers=len(self._als))

    def _run(self, kw):
        al = self._free.get()
        try:
            return al.align(**kw)
        finally:
            self._free.put(al)

    def submit(self, seqA, offA, pairs, k: int, X: int, **kw):
        """Queue one ``Aligner.align`` call; returns a Future of (results, cells)."""
        return self._pool.submit(self._run, dict(seqA=seqA, offA=offA, pairs=pairs, k=k, X=X, **kw))

    def map(self, batches):
        """Align an iterable of ``align`` keyword dicts; results in order."""
        futs = [self._pool.submit(self._run, dict(b)) for b in batches]
        return [f.result() for f in futs]

    def close(self):
        if getattr(self, "_pool", None) is not None:
            self._pool.shutdown(wait=True)
            self._pool = None
            for al in self._als:
                al.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def alu_peaks(device: int = 0) -> dict:
    """xdrop_alu_peaks: measured issue rate of each single-instruction probe on `device` ->
    {probe: {"lane_ops_per_s": .., "inst_per_clk_sm": ..}} (csrc/xdrop_peaks.cu)."""
    out = np.zeros(2 * len(PEAK_PROBES), dtype=np.float64)
    st = N.lib.xdrop_alu_peaks(int(device), out.ctypes.data, out.shape[0])
    N.check(st, "xdrop_alu_peaks")
    return {p: {"lane_ops_per_s": float(out[2 * i]), "inst_per_clk_sm": float(out[2 * i + 1])}
            for i, p in enumerate(PEAK_PROBES)}


def adaptive_filter_device(offA, pairs, out, keep, phi: float, c: float, offB=None, stream=None):
    """xdrop_adaptive_filter_device (f2, reading Q12) on torch CUDA tensors: offsets int64[n+1],
    pairs int32[n,4], out int32[n,5] (alignment results), keep uint8[n] (written)."""
    offB = offA if offB is None else offB
    dev = pairs.device.index
    n = int(pairs.shape[0])
    _check_tensor("offA", offA, (1,), ("int64",), dev)
    _check_tensor("offB", offB, (1,), ("int64",), dev)
    _check_tensor("pairs", pairs, (2,), ("int32",), dev, cols=4)
    _check_tensor("out", out, (2,), ("int32",), dev, rows=n, cols=5)
    _check_tensor("keep", keep, (1,), ("uint8",), dev, rows=n)
    err = ctypes.c_int64(-1)
    s = stream.cuda_stream if stream is not None else None
    st = N.lib.xdrop_adaptive_filter_device(offA.data_ptr(), offA.shape[0] - 1, offB.data_ptr(), offB.shape[0] - 1,
                                            pairs.data_ptr(), out.data_ptr(), n, float(phi), float(c),
                                            keep.data_ptr(), ctypes.byref(err), s)
    if st != N.OK:
        raise XdropError(int(st), "xdrop_adaptive_filter_device", int(err.value))


def seed_kmer_freq_device(seq, off, pairs, k: int, lower: int, upper: int, freq=None, keep=None, stream=None):
    """xdrop_seed_kmer_freq_device (f4) on torch CUDA tensors: ASCII pool uint8, offsets
    int64[n_reads+1], pairs int32[n,4]; fills freq int32[n] and / or keep uint8[n]."""
    dev = pairs.device.index
    n = int(pairs.shape[0])
    _check_tensor("seq", seq, (1,), ("uint8", "int8"), dev)
    _check_tensor("off", off, (1,), ("int64",), dev)
    _check_tensor("pairs", pairs, (2,), ("int32",), dev, cols=4)
    if freq is not None:
        _check_tensor("freq", freq, (1,), ("int32",), dev, rows=n)
    if keep is not None:
        _check_tensor("keep", keep, (1,), ("uint8",), dev, rows=n)
    err = ctypes.c_int64(-1)
    s = stream.cuda_stream if stream is not None else None
    st = N.lib.xdrop_seed_kmer_freq_device(seq.data_ptr(), off.data_ptr(), off.shape[0] - 1, int(seq.shape[0]),
                                           pairs.data_ptr(), n, int(k), int(lower), int(upper),
                                           freq.data_ptr() if freq is not None else None,
                                           keep.data_ptr() if keep is not None else None, ctypes.byref(err), s)
    if st != N.OK:
        raise XdropError(int(st), "xdrop_seed_kmer_freq_device", int(err.value))


def pair_costs(offsets: np.ndarray, pairs: np.ndarray, k: int, offsets_b=None) -> np.ndarray:
    """Estimated cost of each pair (the host scheduler's w): anti-diagonals of
    its two extensions ~ min prefix + min suffix (+1)."""
    pairs = np.asarray(pairs).reshape(-1, 4).astype(np.int64)
    la = np.diff(np.asarray(offsets, dtype=np.int64))
    lb = la if offsets_b is None else np.diff(np.asarray(offsets_b, dtype=np.int64))
    a, b = pairs[:, 0], pairs[:, 1] & 0x7fffffff
    return (np.minimum(pairs[:, 2], pairs[:, 3]) +
            np.minimum(la[a] - pairs[:, 2] - k, lb[b] - pairs[:, 3] - k) + 1)


def shard_pairs(w, n_shards: int):
    """Split pairs over n_shards GPUs by estimated cells with the library's own LPT partitioner (the
    CELLS policy of csrc/sched.cpp, host-only dry run): returns one index array per shard."""
    if n_shards <= 1:
        return [np.arange(np.asarray(w).shape[0])]
    _, _, gpu = sched_simulate(n_shards, "cells", 1, np.asarray(w, dtype=np.int64))
    return [np.nonzero(gpu == s)[0] for s in range(n_shards)]


def _check_tensor(name, t, dims, dtypes, device, rows=None, cols=None):
    """Marshalling guard of align_device: the C ABI reads raw device pointers with fixed layouts
    (include/xdrop.h), so a wrong dtype, shape, stride or device would be misread silently."""
    if t.dim() not in dims:
        raise ValueError(f"{name}: expected {dims[0]}-D tensor, got shape {tuple(t.shape)}")
    if str(t.dtype).replace("torch.", "") not in dtypes:
        raise ValueError(f"{name}: expected dtype {dtypes[0]}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous")
    if t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name}: expected a tensor on cuda:{device}, got {t.device}")
    if rows is not None and t.shape[0] != rows:
        raise ValueError(f"{name}: expected {rows} rows, got {t.shape[0]}")
    if cols is not None and (t.dim() != 2 or t.shape[1] != cols):
        raise ValueError(f"{name}: expected {cols} columns, got shape {tuple(t.shape)}")


def ring_left(rank: int, batch: int, counts) -> int | None:
    """Alg. 1 l.18-24 left-predecessor search (None when the walk returns to rank)."""
    c = np.ascontiguousarray(counts, dtype=np.int32)
    r = N.lib.xdrop_ring_left(rank, batch, c.ctypes.data, c.shape[0])
    return None if r < 0 else r


def ring_right(rank: int, batch: int, counts) -> int | None:
    """Alg. 1 l.26-30 right-successor search."""
    c = np.ascontiguousarray(counts, dtype=np.int32)
    r = N.lib.xdrop_ring_right(rank, batch, c.ctypes.data, c.shape[0])
    return None if r < 0 else r


def sched_simulate(m: int, policy: str, n_ranks: int, w, batch_size: int = 10000, subbatches: int = 1,
                   ns_per_unit: float = 0.0):
    """Host-only dry run of a scheduling policy -> (trace, stats, gpu_of_pair)."""
    w = np.ascontiguousarray(w, dtype=np.int64)
    n = w.shape[0]
    cap = 4 * (n // max(1, batch_size) + 2) * max(1, n_ranks) * max(1, subbatches) * max(1, m) + 64
    trace = np.zeros(cap, dtype=TRACE_DTYPE)
    gpu = np.full(n, -1, dtype=np.int32)
    st = N.SchedStats()
    r = N.lib.xdrop_sched_simulate(m, N.POLICIES[policy], n_ranks, batch_size, subbatches, w.ctypes.data, n,
                                   ns_per_unit, ctypes.byref(st), trace.ctypes.data, cap, gpu.ctypes.data)
    if r < 0:
        raise XdropError(int(r), "xdrop_sched_simulate")
    stats = dict(handoffs=st.handoffs, exchange_msgs=st.exchange_msgs, turns=st.turns, span_ms=st.span_ms,
                 max_concurrent=st.max_concurrent)
    return trace[:min(r, cap)], stats, gpu
