"""N>1 plumbing of bench.py on CPU: world_size-2 gloo (one process per rank).

Pairs shard with no data-path collective: the only collectives
are the max-over-ranks time and the cell/pair sums, which these tests exercise.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tmax = bench.allreduce(10.0 + rank, "max", world)
    csum = bench.allreduce(100.0 * (rank + 1), "sum", world)
    bench.barrier(world)

    class A:
        config, scale, X = "tiny", 1.0, None
    w = bench.shard_workload(A, rank)
    out.put((rank, tmax, csum, int(w.pairs[:, 2].sum()), w.recipe["seed"]))
    dist.destroy_process_group()


def test_gloo_reductions_and_distinct_shards():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert [r[1] for r in res] == [11.0, 11.0]          # max over ranks
    assert [r[2] for r in res] == [300.0, 300.0]        # sum over ranks
    assert res[0][4] != res[1][4]                       # each rank owns its own seeded shard
    assert res[0][3] != res[1][3]


@pytest.mark.slow
def test_torchrun_reference_arm_two_ranks():
    """`bench.py --impl reference` under torchrun: rank 0 prints one JSON line, rank 1 exits 0."""
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "tiny",
           "--cpu-seconds", "0.2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GCUPS" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["ms_per_step"] > 0 and "sample_s" not in d["cpu_baseline"]


def test_strong_shards_lpt_balance():
    """bench.py --scaling strong: the same global batch split over ranks by the library's LPT on
    estimated cells; shards are disjoint, cover every pair, and the LPT bound holds: the heaviest
    shard exceeds the mean by at most the largest single item (PAPER.md:115-118 one2all splits a
    batch over all GPUs; here by cost)."""
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2309_07270_b200 as xd
    from synth import workload as W
    w = W.config("cfg1")
    cost = xd.pair_costs(w.offsets, w.pairs, w.k)
    for n in (2, 3, 8):
        sh = xd.shard_pairs(cost, n)
        allidx = np.sort(np.concatenate(sh))
        assert np.array_equal(allidx, np.arange(w.n_pairs))
        loads = np.array([cost[s].sum() for s in sh])
        assert loads.max() - loads.mean() <= cost.max()


def _strong_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class A:
        config, scale, X, scaling = "tiny", 1.0, None, "strong"
    w, idx = bench.rank_workload(A, rank, world)
    out.put((rank, w.recipe["seed"], idx.tolist(), int(w.n_pairs)))
    dist.destroy_process_group()


def test_gloo_strong_scaling_shards():
    """Under gloo with world_size 2, --scaling strong gives both ranks the SAME seeded batch and
    disjoint LPT shards of it that together cover every pair."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_strong_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert res[0][1] == res[1][1]                        # one global batch
    a, b = set(res[0][2]), set(res[1][2])
    assert not (a & b) and len(a | b) == res[0][3]


def _gather_worker(rank, world, port, out):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 11
    idx = np.arange(rank, n, world)                      # disjoint shards of a global batch
    res = torch.from_numpy(np.stack([idx * 10 + j for j in range(5)], axis=1).astype(np.int32))
    cells = torch.from_numpy((idx * 1000).astype(np.int64))
    g, c = bench.gather_results(res, cells, idx, n, world)
    out.put((rank, g.numpy().tolist(), c.numpy().tolist()))
    dist.destroy_process_group()


def test_gloo_strong_result_gather():
    """--scaling strong's result gather (optional): every rank ends with the whole
    batch's results in pair order, shards of unequal size included."""
    import numpy as np
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(3))
    want = [[10 * i + j for j in range(5)] for i in range(11)]
    for _, g, c in res:
        assert g == want and c == [1000 * i for i in range(11)]
