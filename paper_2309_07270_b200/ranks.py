"""Multi-process rank mode: the paper's GPU schedulers with real OS
processes as the MPI ranks (§III, Alg. 1).

Each process is one logical rank.  It owns an equal contiguous chunk of the pair list
(PAPER.md:80), splits it into batches of ``batch_size`` pairs and ``c`` sub-batches
(PAPER.md:100), exchanges batch counts with its ring (Alg. 1 l.5-11) and then takes GPU
turns gated by a token passed with point-to-point messages (Alg. 1 l.18-30; blocking,
source-matched receives, as MPI_Recv).  The token order is reading Q21:
Alg. 1's ring within a batch level, and at the wrap-around that ends a level, the first
member of the next level (Alg. 1 read literally deadlocks on counts such as [2, 2, 1]).

Policies: ``one2all`` (one global ring; the holder aligns its sub-batch on all of its
devices), ``one2one`` (ring of the ranks r = g mod m; token per sub-batch) and
``opt_one2one`` (the same rings, token per batch; BASELINE's "mixed scheme").

The alignment itself always goes through the C ABI (``Aligner``); this module only
orchestrates processes.  ``verify`` re-checks a gathered trace against the scheduler
invariants of SPEC.md:302-311 (mutual exclusion per GPU, exactly-once, per-rank order,
ring order, one2all global serialisation) using the trace alone.
"""
from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np

POLICIES = ("one2all", "one2one", "opt_one2one")


# ------------------------------------------------------------------ partitioning
def rank_chunk(n_pairs: int, n_ranks: int, rank: int) -> tuple[int, int]:
    """Equal contiguous chunk of rank (remainder to the lowest ranks)."""
    base, extra = divmod(n_pairs, n_ranks)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def subbatches(lo: int, hi: int, batch_size: int, c: int) -> list[list[np.ndarray]]:
    """Batches of batch_size pairs, each split into c near-equal sub-batches, larger
    first.  Empty sub-batches are KEPT as no-op turns (reading Q22)."""
    out = []
    for b0 in range(lo, hi, batch_size):
        bs = min(batch_size, hi - b0)
        subs, q = [], b0
        for s in range(c):
            ss = bs // c + (1 if s < bs % c else 0)
            subs.append(np.arange(q, q + ss, dtype=np.int64))
            q += ss
        out.append(subs)
    return out


# ----------------------------------------------------------------- token order
@dataclass
class Ring:
    """Reading Q21's token order over one ring; the order itself is the C library's
    (xdrop_ring_turn_next / _prev, csrc/sched.cpp), the one the in-process scheduler uses."""
    members: list[int]          # rank ids, ascending
    counts: list[int]           # batches per member
    turns_per_batch: int        # c (per sub-batch token) or 1 (per batch token)

    def _counts(self):
        import ctypes
        return (ctypes.c_int * len(self.counts))(*[int(x) for x in self.counts])

    def next(self, u: int, b: int, it: int) -> int:
        """Member index owning the turn after (b, it, u); -1 if none (reading Q21)."""
        from . import _native as N
        return int(N.lib.xdrop_ring_turn_next(u, b, it, self._counts(), len(self.counts), self.turns_per_batch,
                                              None, None))

    def prev(self, u: int, b: int, it: int) -> int:
        from . import _native as N
        return int(N.lib.xdrop_ring_turn_prev(u, b, it, self._counts(), len(self.counts), self.turns_per_batch))


def ring_of(policy: str, rank: int, n_ranks: int, m: int) -> list[int]:
    if policy == "one2all":
        return list(range(n_ranks))
    return [r for r in range(n_ranks) if r % m == rank % m]          # PAPER.md:186 "n mod m"


# ---------------------------------------------------------------- messaging
class Comm:
    """Point-to-point messages; the default uses torch.distributed (gloo/nccl-free)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.dist, self.torch, self.group = dist, torch, group
        self.sent = 0

    def send(self, dst: int, value: int):
        self.dist.send(self.torch.tensor([value], dtype=self.torch.int64), dst=dst, group=self.group)
        self.sent += 1

    def recv(self, src: int) -> int:
        t = self.torch.zeros(1, dtype=self.torch.int64)
        self.dist.recv(t, src=src, group=self.group)
        return int(t.item())


@dataclass
class Turn:
    rank: int
    gpu: int
    batch: int
    sub: int
    n_pairs: int
    t0: float
    t1: float


@dataclass
class RankResult:
    rank: int
    turns: list = field(default_factory=list)
    handoffs: int = 0
    exchange_msgs: int = 0
    pair_index: np.ndarray = None


def run_rank(rank: int, n_ranks: int, policy: str, m: int, n_pairs: int, batch_size: int, c: int,
             comm, runner, clock=time.monotonic) -> RankResult:
    """One rank's whole schedule.  runner(gpu_slots, idx) aligns pairs idx on the given
    device slots (all m for one2all, rank mod m otherwise) and returns when done; it may return
    {slot: (t0, t1)} with each device's own busy interval (one2all runs its devices concurrently),
    else every slot's turn spans the whole call."""
    if policy not in POLICIES:
        raise ValueError(policy)
    lo, hi = rank_chunk(n_pairs, n_ranks, rank)
    work = subbatches(lo, hi, batch_size, c)
    members = ring_of(policy, rank, n_ranks, m)
    u = members.index(rank)
    res = RankResult(rank, pair_index=np.arange(lo, hi))
    # Alg. 1 l.5-11: every ring member sends its batch count to every other member
    counts = [0] * len(members)
    counts[u] = len(work)
    sent0 = comm.sent
    for v, r in enumerate(members):
        if r == rank:
            for w in members:
                if w != rank:
                    comm.send(w, len(work))
        else:
            counts[v] = comm.recv(r)
    res.exchange_msgs = comm.sent - sent0
    opt = policy == "opt_one2one"
    ring = Ring(members, counts, 1 if opt else c)
    slots = list(range(m)) if policy == "one2all" else [rank % m]
    sent0 = comm.sent
    for b in range(1, len(work) + 1):
        for it in range(1, (1 if opt else c) + 1):
            pv = ring.prev(u, b, it)
            if pv >= 0 and pv != u:
                comm.recv(members[pv])                                   # l.18-24: implicit barrier
            subs = work[b - 1] if opt else [work[b - 1][it - 1]]
            for s_i, idx in enumerate(subs):
                sub_no = (s_i + 1) if opt else it
                t0 = clock()
                per = runner(slots, idx) if idx.size else None
                t1 = clock()
                for g in slots:
                    g0, g1 = per[g] if per and g in per else (t0, t1)
                    res.turns.append(Turn(rank, g, b, sub_no, int(idx.size), g0, g1))
            nx = ring.next(u, b, it)
            if nx >= 0 and nx != u:
                comm.send(members[nx], 1)                                # l.26-30
    res.handoffs = comm.sent - sent0
    return res


# -------------------------------------------------------------------- verify
def verify(turns: list[Turn], n_pairs: int, n_ranks: int, m: int, policy: str, batch_size: int,
           c: int, eps: float = 0.0) -> list[str]:
    """Trace-only checks.  Returns violations (empty = pass)."""
    bad = []
    # mutual exclusion per GPU (one2all: across all GPUs, one turn at a time)
    by_gpu = {}
    for t in turns:
        by_gpu.setdefault(t.gpu, []).append(t)
    for g, ev in by_gpu.items():
        ev = sorted(ev, key=lambda t: t.t0)
        for a, b in zip(ev, ev[1:]):
            if b.t0 < a.t1 - eps:
                bad.append(f"overlap on gpu {g}: rank {a.rank} b{a.batch}s{a.sub} and rank {b.rank} b{b.batch}s{b.sub}")
    if policy == "one2all":
        per_turn = {}
        for t in turns:
            key = (t.rank, t.batch, t.sub)
            lo, hi = per_turn.get(key, (t.t0, t.t1))
            per_turn[key] = (min(lo, t.t0), max(hi, t.t1))
        iv = sorted(per_turn.items(), key=lambda kv: kv[1][0])
        for (ka, a), (kb, b) in zip(iv, iv[1:]):
            if b[0] < a[1] - eps:
                bad.append(f"one2all: turns {ka} and {kb} overlap")
    else:
        for t in turns:
            if t.gpu != t.rank % m:
                bad.append(f"affinity: rank {t.rank} used gpu {t.gpu}")
    # exactly once: the (rank, batch, sub) multiset equals the partition (sizes included)
    seen = {}
    for t in turns:
        key = (t.rank, t.batch, t.sub)
        if policy == "one2all":                 # one entry per device slot of the same turn
            seen[key] = max(seen.get(key, 0), t.n_pairs)
        else:
            if key in seen:
                bad.append(f"duplicate turn {key}")
            seen[key] = t.n_pairs
    for r in range(n_ranks):
        lo, hi = rank_chunk(n_pairs, n_ranks, r)
        for b, subs in enumerate(subbatches(lo, hi, batch_size, c), start=1):
            for s, idx in enumerate(subs, start=1):
                if idx.size and seen.get((r, b, s)) != idx.size:
                    bad.append(f"missing or wrong turn r{r}.b{b}.s{s}")
    # per-rank order: (batch, sub) lexicographic in time
    for r in range(n_ranks):
        ev = sorted([t for t in turns if t.rank == r], key=lambda t: t.t0)
        keys = [(t.batch, t.sub) for t in ev]
        if keys != sorted(keys):
            bad.append(f"rank {r} out of order")
    # ring order (token sequence): within each ring, turns follow (batch, iteration, rank)
    rings = {}
    for t in turns:
        rid = 0 if policy == "one2all" else t.rank % m
        rings.setdefault(rid, {})
        it = 1 if policy == "opt_one2one" else t.sub
        rings[rid].setdefault((t.rank, t.batch, it), t.t0)
    for rid, d in rings.items():
        by_time = [k for k, _ in sorted(d.items(), key=lambda kv: kv[1])]
        expected = sorted(d.keys(), key=lambda k: (k[1], k[2], k[0]))
        if by_time != expected:
            bad.append(f"ring {rid}: token order {by_time[:6]} != {expected[:6]}")
    return bad


def metrics(turns: list[Turn], results: list[RankResult]) -> dict:
    """Table I-style metrics: alignment span, handoff / exchange message counts."""
    t0 = min((t.t0 for t in turns), default=0.0)
    t1 = max((t.t1 for t in turns), default=0.0)
    return dict(span_ms=(t1 - t0) * 1e3, handoffs=sum(r.handoffs for r in results),
                exchange_msgs=sum(r.exchange_msgs for r in results), turns=len(turns))


# ------------------------------------------------------------ process driver
def _worker(rank, n_ranks, port, policy, m, batch_size, c, w_arrays, params, use_gpu, sleep_ns_per_pair, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=n_ranks)
    seq, off, pairs = w_arrays
    n_pairs = pairs.shape[0]
    out = np.zeros((n_pairs, 5), dtype=np.int32)
    cells = np.zeros(n_pairs, dtype=np.int64)
    if use_gpu:
        from . import Aligner
        slots = list(range(m)) if policy == "one2all" else [rank % m]
        ndev = torch.cuda.device_count()
        devs = {g: torch.device(f"cuda:{g % ndev}") for g in slots}
        als = {g: Aligner(devices=[g % ndev]) for g in slots}
        res_seq = {g: torch.from_numpy(seq).to(devs[g]) for g in slots}         # pool resident per device
        res_off = {g: torch.from_numpy(off).to(devs[g]) for g in slots}
        dpairs = {g: torch.from_numpy(pairs).to(devs[g]) for g in slots}

        def run_part(g, part, times):
            t0 = time.monotonic()
            dev = devs[g]
            sub = dpairs[g][torch.from_numpy(part).to(dev)]
            o = torch.zeros((part.size, 5), dtype=torch.int32, device=dev)
            cl = torch.zeros(part.size, dtype=torch.int64, device=dev)
            als[g].align_device(res_seq[g], res_off[g], sub, o, cl, **params)   # ctypes drops the GIL
            out[part] = o.cpu().numpy()
            cells[part] = cl.cpu().numpy()
            times[g] = (t0, time.monotonic())

        def runner(gs, idx):
            # one2all: the holder splits its sub-batch over its devices and drives them CONCURRENTLY
            # (one host thread per device), each turn timed on its own device
            parts = [(g, p) for g, p in zip(gs, np.array_split(idx, len(gs))) if p.size]
            times = {}
            if len(parts) == 1:
                run_part(parts[0][0], parts[0][1], times)
                return times
            errs = []

            def body(g, p):
                try:
                    torch.cuda.set_device(devs[g])
                    run_part(g, p, times)
                except BaseException as e:      # noqa: BLE001 (re-raised below)
                    errs.append(e)
            ths = [threading.Thread(target=body, args=gp) for gp in parts]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            if errs:
                raise errs[0]
            return times
    else:
        def runner(gs, idx):
            time.sleep(sleep_ns_per_pair * idx.size * 1e-9)
    res = run_rank(rank, n_ranks, policy, m, n_pairs, batch_size, c, Comm(), runner)
    lo, hi = rank_chunk(n_pairs, n_ranks, rank)
    q.put((rank, [t.__dict__ for t in res.turns], res.handoffs, res.exchange_msgs, lo, hi, out[lo:hi], cells[lo:hi]))
    dist.barrier()
    dist.destroy_process_group()


def spawn(n_ranks: int, policy: str, m: int, seq: np.ndarray, off: np.ndarray, pairs: np.ndarray,
          batch_size: int = 10000, c: int = 1, params: dict | None = None, use_gpu: bool = True,
          sleep_ns_per_pair: float = 0.0, port: int | None = None, timeout: float = 600.0):
    """Run the schedule with n_ranks OS processes; returns (results, cells, turns, metrics, violations)."""
    import socket
    import torch.multiprocessing as mp
    if port is None:
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    arrays = (np.ascontiguousarray(seq), np.ascontiguousarray(off), np.ascontiguousarray(pairs, dtype=np.int32))
    procs = [ctx.Process(target=_worker, args=(r, n_ranks, port, policy, m, batch_size, c, arrays, params or {},
                                               use_gpu, sleep_ns_per_pair, q)) for r in range(n_ranks)]
    for p in procs:
        p.start()
    got = [q.get(timeout=timeout) for _ in range(n_ranks)]
    for p in procs:
        p.join(timeout)
        if p.exitcode != 0:
            raise RuntimeError(f"rank process exited with {p.exitcode}")
    n = pairs.shape[0]
    out = np.zeros((n, 5), dtype=np.int32)
    cells = np.zeros(n, dtype=np.int64)
    turns, results = [], []
    for rank, tl, h, ex, lo, hi, o, cl in got:
        out[lo:hi] = o
        cells[lo:hi] = cl
        turns += [Turn(**t) for t in tl]
        results.append(RankResult(rank, handoffs=h, exchange_msgs=ex))
    bad = verify(turns, n, n_ranks, m, policy, batch_size, c)
    return out, cells, turns, metrics(turns, results), bad
