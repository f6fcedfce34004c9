#!/usr/bin/env python3
"""Benchmark of the batched X-drop hot path (BASELINE.json metric: GCUPS and alignments/s).

One step = one pass of the whole hot path over one batch:
ASCII->2-bit pack, validation + cost estimate + length-sorted queue, left/right
band kernels (all escalation levels), combine -- through the C ABI
(xdrop_align_batch_device) on inputs resident in HBM.  ``e2e`` repeats the
measurement through xdrop_align_batch with pinned HOST buffers (H2D of the read
pool + pairs and D2H of the results inside the timed region).

Launch: python bench.py [--gpus N --steps K --warmup W] (N>1 under torchrun,
one rank per GPU; pairs are independent, each rank aligns its own shard:
weak scaling, no data-path collective).  ``--impl reference`` times the CPU
oracle (the only other place this file executes oracle/).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_OPS_PER_CELL = 8          # algorithmic INT32 ops per DP cell
SM_COUNT_NOMINAL = 148


# one metric string for both arms (the driver divides the native line by the reference line)
METRIC = "GCUPS (X-drop DP cells per second; also alignments/s, INT32 roofline fraction)"

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="ecoli", help="synth.workload config (BASELINE configs[1] = ecoli)")
    ap.add_argument("--scale", type=float, default=1.0, help="pair-count scale (tests only)")
    ap.add_argument("--X", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-compat", action="store_true", help="skip the compat-mode (XDROP_FLAG_SEQAN_COMPAT) entry")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the bounded oracle sample")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = each rank its own seeded batch of the config; strong = ONE global batch "
                         "split over the ranks by estimated cells (the library's LPT, BASELINE configs[2])")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the ncu child run that measures the dominant kernel's DRAM bytes per launch")
    return ap.parse_args()


# --------------------------------------------------------------------------- dist
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def allreduce(x: float, op: str, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def allgather(x: float, world: int, device=None) -> list:
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(o.item()) for o in out]


def gather_results(out, cells, idx, n_total, world, device=None):
    """--scaling strong: the optional result gather of SURVEY.md §8(e) (24 B per pair over NCCL, or gloo
    on CPU).  Every rank contributes its shard's (n, 5) int32 results and int64 cells at the pair
    indices `idx` it aligned; returns the global (n_total, 5) / (n_total,) arrays on every rank."""
    import torch
    if world == 1:
        return out, cells
    import torch.distributed as dist
    n_my = torch.tensor([int(idx.shape[0])], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n_my) for _ in range(world)]
    dist.all_gather(sizes, n_my)
    cap = int(max(int(x.item()) for x in sizes))
    pad = torch.full((cap, 7), -1, dtype=torch.int64, device=device)
    k = int(idx.shape[0])
    if k:
        pad[:k, 0] = torch.as_tensor(idx, dtype=torch.int64, device=device)
        pad[:k, 1:6] = out.to(device=device, dtype=torch.int64)
        pad[:k, 6] = cells.to(device=device, dtype=torch.int64)
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    full = torch.cat(parts, 0)
    full = full[full[:, 0] >= 0]
    g_out = torch.zeros((n_total, 5), dtype=torch.int32, device=device)
    g_cells = torch.zeros(n_total, dtype=torch.int64, device=device)
    g_out[full[:, 0]] = full[:, 1:6].to(torch.int32)
    g_cells[full[:, 0]] = full[:, 6]
    return g_out, g_cells


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------------- workload
def shard_workload(args, rank):
    """Each rank aligns its own synthetic batch of the named config (seed offset by rank)."""
    from synth import workload as W
    base = {"cfg1": 1, "ecoli": 2, "xsweep": 4, "celegans": 5, "tiny": 7}[args.config]
    return W.config(args.config, scale=args.scale, X=args.X, seed=base + 1000 * rank)


def rank_workload(args, rank, world):
    """(workload, pair indices this rank aligns).  weak: its own seeded batch, every pair; strong: the
    rank-0 seed's batch for every rank and this rank's shard of it (paper_2309_07270_b200.shard_pairs:
    LPT over estimated cells, the same partitioner as the library's CELLS policy)."""
    if getattr(args, "scaling", "weak") != "strong" or world == 1:
        w = shard_workload(args, rank)
        return w, np.arange(w.n_pairs)
    import paper_2309_07270_b200 as xd
    w = shard_workload(args, 0)
    sh = xd.shard_pairs(xd.pair_costs(w.offsets, w.pairs, w.k), world)
    return w, sh[rank]


def workload_desc(w, args, world):
    lens = np.diff(w.offsets)
    return {"workload": f"{w.name} (BASELINE configs[1]: E. coli-shaped, ~10 kb PacBio-like reads, 15% error)"
            if args.config == "ecoli" else w.name,
            "pairs_per_gpu": w.n_pairs if args.scaling == "weak" else round(w.n_pairs / world, 1),
            "global_pairs": w.n_pairs * world if args.scaling == "weak" else w.n_pairs,
            "reads_per_gpu": int(lens.shape[0]),
            "mean_read_len": round(float(lens.mean()), 1), "pool_bases_per_gpu": int(w.offsets[-1]),
            "k": w.k, "X": w.X, "scoring": [w.M, w.mu, w.g],
            "errors": "1.5% sub / 9% ins / 4.5% del", "parallelism": f"dp{world} (independent shards)" if args.scaling == "weak" else
            f"dp{world} (one batch split by estimated cells, LPT)",
            "l2": "flushed between timed steps (256 MiB memset)", "recipe_seed": w.recipe.get("seed")}


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            cmd = ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                   "-lms", "50"]
            if shutil.which("stdbuf"):             # line-buffered, or samples are lost on terminate
                cmd = ["stdbuf", "-oL"] + cmd
            self.proc = subprocess.Popen(cmd, stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.f:
            return None
        try:
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        finally:
            try:
                os.unlink(self.f.name)
            except Exception:
                pass
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 8]
        if not rows:
            return None
        sm = np.array([float(r[0]) for r in rows])
        load = sm[sm > 0.5 * sm.max()] if sm.size else sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": int(sm.size), "power_w_max": max(float(r[2]) for r in rows)}


# ------------------------------------------------------------------- ncu traffic
# ncu kernel-name regex of the dominant band kernel (stats()["band_kernel"])
DOM_REGEX = {"tiered": "pk_tiered_kernel", "shared": "pk_merged_kernel", "merged32": "band_merged_kernel"}


def ncu_traffic(args, kregex):
    """DRAM bytes (read + write) of ONE launch of the dominant kernel, measured by ncu in a child run
    of this same benchmark (same config; the launch profiled is the first timed step's, after the L2
    flush).  Returns (bytes or None, note).  Numbers printed by the child are never used as bench values."""
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu is None:
        return None, "ncu not found"
    warm = 3
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", f"regex:{kregex}", "--launch-skip", str(warm), "--launch-count", "1",
           "--csv", sys.executable, os.path.abspath(__file__), "--steps", "1", "--warmup", str(warm),
           "--no-e2e", "--no-cpu", "--no-traffic", "--no-compat", "--config", args.config, "--scale", str(args.scale)]
    if args.X is not None:
        cmd += ["--X", str(args.X)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    except Exception as e:          # noqa: BLE001
        return None, f"ncu child failed: {type(e).__name__}"
    vals = {}
    import csv
    import io
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    for row in csv.reader(io.StringIO("\n".join(rows))):
        if len(row) >= 3 and row[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            unit, val = row[-2], float(row[-1].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                     "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
                     "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1)
            vals[row[-3]] = val * scale
    if "dram__bytes_read.sum" not in vals:
        return None, f"ncu gave no DRAM metrics (rc {r.returncode}): {(r.stdout + r.stderr)[-300:]!r}"
    b = int(vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0))
    return b, (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum on launch {warm + 1} of {kregex} "
               f"(first timed step, after the L2 flush) in a child run of this config; "
               f"read {int(vals['dram__bytes_read.sum'])} B, write {int(vals.get('dram__bytes_write.sum', 0))} B, "
               f"{vals.get('gpu__time_duration.sum', 0):.3f} ms under ncu (not a bench value)")


# ---------------------------------------------------------------------- cpu legs
def cpu_info():
    """Host CPU model, logical threads and physical cores (for the cpu_baseline / reference lines)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:
        phys = None
    return {"cpu_model": model, "logical_cpus": os.cpu_count() or 1, "physical_cores": phys}


def oracle_sample(w, seconds: float, rng_seed: int = 0):
    """Bounded sample of the workload for the oracle: a pilot fixes the rate, then an
    evenly spaced sample of pairs sized to ~`seconds` of CPU work is timed.  Returns the
    baseline dict and (idx, results, cells) of the sample (bench.py checks the GPU against them)."""
    import oracle
    n = w.n_pairs
    ci = cpu_info()
    cores = ci["logical_cpus"]
    pilot = np.arange(0, n, max(1, n // 64))[:64]
    t = time.perf_counter()
    _, c = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs[pilot], w.k, w.M, w.mu, w.g, w.X,
                              nthreads=cores)
    dt = max(1e-3, time.perf_counter() - t)
    per_pair = dt / pilot.size
    m = int(min(n, max(pilot.size, seconds / per_pair)))
    idx = np.linspace(0, n - 1, m).astype(np.int64)
    t = time.perf_counter()
    res, cells = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, w.pairs[idx], w.k, w.M, w.mu, w.g, w.X,
                                    nthreads=cores)
    dt = time.perf_counter() - t
    mcells = float(cells.sum()) / dt / 1e6
    base = {"value": round(mcells / 1e3, 4), "unit": "GCUPS", "cores": cores, "kind": "oracle",
            "sample": f"{m} of {n} pairs (evenly spaced), {int(cells.sum())} cells in {dt:.2f} s "
                      f"on {cores} host threads; alignments/s {m / dt:.1f}",
            "threads_used": cores, "cpu_model": ci["cpu_model"], "physical_cores": ci["physical_cores"],
            "mcells_per_s_per_thread": round(mcells / cores, 2),
            "mcells_per_s_per_physical_core": round(mcells / ci["physical_cores"], 2) if ci["physical_cores"] else None,
            "alignments_per_s": round(m / dt, 2), "sample_s": round(dt, 4), "sample_pairs": m}
    return base, (idx, res, cells)


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle as it stands, rank 0 only."""
    if rank != 0:
        return
    w = shard_workload(args, 0)
    vals = []
    t_run = time.perf_counter()
    for step in range(args.warmup + args.steps):
        r, _ = oracle_sample(w, seconds=max(2.0, min(args.cpu_seconds, 120.0 / max(1, args.steps + args.warmup))))
        if step >= args.warmup:
            vals.append(r)
    run_s = time.perf_counter() - t_run
    v = float(np.median([r["value"] for r in vals]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GCUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": workload_desc(w, args, world),
            # one step = one bounded oracle sample of the workload (the time actually spent, not extrapolated)
            "ms_per_step": round(float(np.median([r["sample_s"] for r in vals])) * 1e3, 3),
            "ms_per_step_note": "measured wall time of one step = one bounded, evenly spaced oracle sample of the "
                                "batch (sample size in cpu_baseline.sample); value = that sample's cells / time",
            "run_s": round(run_s, 2),
            "cpu_baseline": {k: x for k, x in {**vals[-1], "value": v}.items()
                             if k not in ("sample_s", "sample_pairs")},
            "e2e": {"value": v, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "alignments_per_s": float(np.median([r["alignments_per_s"] for r in vals]))}
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


# ----------------------------------------------------------------------- native
def run_native(args, world, rank, local):
    import torch
    import paper_2309_07270_b200 as xd

    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    w, sidx = rank_workload(args, rank, world)
    my_pairs = np.ascontiguousarray(w.pairs[sidx])
    n_my = int(my_pairs.shape[0])
    al = xd.Aligner(devices=[local])
    stream = torch.cuda.current_stream(dev)

    # inputs resident in HBM (value); pinned host copies (e2e)
    seq_d = torch.from_numpy(w.seq).to(dev)
    off_d = torch.from_numpy(w.offsets).to(dev)
    pairs_d = torch.from_numpy(my_pairs).to(dev)
    out_d = torch.zeros((n_my, 5), dtype=torch.int32, device=dev)
    cells_d = torch.zeros(n_my, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2

    def step():
        al.align_device(seq_d, off_d, pairs_d, out_d, cells_d, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g, stream=stream)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    step_ms, l0_ms, stats = [], [], []
    with ClockSampler(local) as clk:          # clocks over warm-up + timed steps (same load)
        for _ in range(max(3, args.warmup)):
            step()
        torch.cuda.synchronize(dev)
        cells_step = int(cells_d.sum().item())
        barrier(world)
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.zero_()                                   # untimed L2 flush between timed steps
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            st = al.stats()
            stats.append(st)
        torch.cuda.synchronize(dev)
    barrier(world)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    total_ms_max = allreduce(total_ms, "max", world, dev)
    cells_all = allreduce(float(cells_step * args.steps), "sum", world, dev)
    pairs_all = allreduce(float(n_my * args.steps), "sum", world, dev)
    per_gpu_ms = allgather(total_ms / args.steps, world, dev)
    gcups = cells_all / (total_ms_max * 1e-3) / 1e9
    aps = pairs_all / (total_ms_max * 1e-3)

    # dominant kernel: band level 0 (lane per extension)
    lvl_ms = np.mean([s["level_ms"] for s in stats], axis=0)
    lvl_cells = stats[-1]["level_cells"]
    dom = int(np.argmax(lvl_ms))
    band_kernel = stats[-1].get("band_kernel", "tiered")
    dom_names = [{"tiered": "xk::pk_tiered_kernel<4,8> (T0 packed 16x2 lane/4-lane modes + T1/T2 in-kernel escalation)",
                  "shared": "xk::pk_merged_kernel<4,8> (one run-time-G packed loop for T0/T1/T2 + 4-lane units)",
                  "merged32": "xk::band_merged_kernel<32,4,8> (32-bit cells)"}[band_kernel],
                 "(merged into level 0)",
                 "xk::band_kernel<32,32> (warp/extension)", "xk::general_kernel"]
    achieved_ops = lvl_cells[dom] * ALGO_OPS_PER_CELL / (lvl_ms[dom] * 1e-3)
    # algorithmic bytes of one band-kernel launch: the 2-bit pool read once
    # (0.25 B/base) + per extension its queue entry (4 B), pair descriptor (16 B), two read offsets
    # pairs (32 B) and its result record (32 B)
    algo_bytes = int(w.offsets[-1]) // 4 + 2 * n_my * (4 + 16 + 32 + 32)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clocks = clk.summary()
    sm_max = (clocks or {}).get("sm_max_mhz") or 1965.0
    # roofline denominators MEASURED on this device (csrc/xdrop_peaks.cu, single-instruction probes,
    # SASS checked by tests/test_capi_host.py::test_peak_probes_sass): the T0 cells are packed 16-bit
    # pairs, so the line's dtype (i16) peak is the VIMNMX3.S16x2 probe's lane-op rate x 2 16-bit ops;
    # the int32 figure (VIMNMX3 probe) is kept beside it
    pk = xd.alu_peaks(local)
    p16 = 2.0 * pk["VIMNMX3.S16x2"]["lane_ops_per_s"]
    p32 = pk["VIMNMX3"]["lane_ops_per_s"]
    nominal32 = sms * 4 * 16 * sm_max * 1e6
    traffic = None
    traffic_note = None
    if not args.no_traffic and world == 1:
        traffic, traffic_note = ncu_traffic(args, DOM_REGEX[band_kernel])
    roofline = {"bound": "alu", "achieved": round(achieved_ops / 1e9, 1), "peak": round(p16 / 1e9, 1),
                "unit": "Gop/s", "frac": round(achieved_ops / p16, 4), "traffic": traffic,
                "peak_basis": "measured: 2 x the thread-instruction rate of the VIMNMX3.S16x2 probe "
                              f"({pk['VIMNMX3.S16x2']['inst_per_clk_sm']:.1f} warp-inst/clk/SM) = 16-bit "
                              "ALU-pipe ops/s (dtype i16: two cells per lane-op)",
                "int32": {"peak": round(p32 / 1e9, 1), "frac": round(achieved_ops / p32, 4),
                          "basis": f"measured VIMNMX3 (32-bit) probe, {pk['VIMNMX3']['inst_per_clk_sm']:.1f} "
                                   "warp-inst/clk/SM"},
                "nominal": {"int32_peak": round(nominal32 / 1e9, 1), "i16x2_peak": round(2 * nominal32 / 1e9, 1),
                            "basis": f"{sms} SMs x 4 SMSP x 16 lanes/clk x {sm_max:.0f} MHz"},
                "probes": {k: {"gops": round(v["lane_ops_per_s"] / 1e9, 1),
                               "inst_per_clk_sm": round(v["inst_per_clk_sm"], 2)} for k, v in pk.items()},
                "kernel": dom_names[dom], "kernel_ms": round(float(lvl_ms[dom]), 3),
                "kernel_share_of_step": round(float(lvl_ms[dom]) / (total_ms / args.steps), 4),
                "ops_per_cell": ALGO_OPS_PER_CELL, "cells_per_launch": int(lvl_cells[dom]),
                "algorithmic_bytes_per_launch": int(algo_bytes),
                "traffic_note": traffic_note}

    # e2e through the host API (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        seq_h = torch.from_numpy(w.seq).pin_memory().numpy()
        off_h = torch.from_numpy(w.offsets).pin_memory().numpy()
        pairs_h = torch.from_numpy(my_pairs).pin_memory().numpy()
        al.align(seq_h, off_h, pairs_h, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)     # warm
        barrier(world)
        t0 = time.perf_counter()
        e_steps = max(1, args.steps)
        for _ in range(e_steps):
            res_h, cells_h = al.align(seq_h, off_h, pairs_h, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)
        e_ms = (time.perf_counter() - t0) * 1e3
        e_ms_max = allreduce(e_ms, "max", world, dev)
        e_cells = allreduce(float(int(cells_h.sum()) * e_steps), "sum", world, dev)
        h2d = int(w.seq.nbytes + w.offsets.nbytes + my_pairs.nbytes)
        d2h = int(n_my * (20 + 8))
        e2e = {"value": round(e_cells / (e_ms_max * 1e-3) / 1e9, 3), "unit": "GCUPS", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e_steps, "ms_per_step": round(e_ms_max / e_steps, 3)}
        # e2e results must equal the device path's
        o = out_d.cpu().numpy()
        assert np.array_equal(o[:, 0], res_h["score"]) and np.array_equal(cells_h, cells_d.cpu().numpy())
        # the same with the read pool registered once (untimed; ELBA aligns batches
        # against the same reads): per step only the pairs go in and the results come out
        pid = al.register_pool(seq_h, off_h)
        al.align_pooled(pid, pairs_h, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)       # warm
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(e_steps):
            res_p, cells_p = al.align_pooled(pid, pairs_h, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)
        p_ms = allreduce((time.perf_counter() - t0) * 1e3, "max", world, dev)
        al.release_pool(pid)
        assert np.array_equal(res_p, res_h) and np.array_equal(cells_p, cells_h)
        e2e["pooled"] = {"value": round(e_cells / (p_ms * 1e-3) / 1e9, 3), "unit": "GCUPS",
                         "h2d_bytes_per_step": int(my_pairs.nbytes), "d2h_bytes_per_step": d2h,
                         "ms_per_step": round(p_ms / e_steps, 3),
                         "note": "xdrop_align_pooled: pool registered (uploaded + packed) once, untimed"}
        # a serving loop: the same host-API call with several batches in flight (xd.Pipeline: one
        # context and host thread per in-flight batch); every step still uploads its pool and pairs
        # and reads its results back inside the timed region
        n_fl = 3
        job = dict(seqA=seq_h, offA=off_h, pairs=pairs_h, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g)
        with xd.Pipeline(n_inflight=n_fl, devices=[local]) as pl:
            pl.map([job] * n_fl)                                                   # warm every context
            barrier(world)
            t0 = time.perf_counter()
            outs = pl.map([job] * e_steps)
            q_ms = allreduce((time.perf_counter() - t0) * 1e3, "max", world, dev)
        assert all(np.array_equal(r, res_h) and np.array_equal(c, cells_h) for r, c in outs)
        e2e["pipelined"] = {"value": round(e_cells / (q_ms * 1e-3) / 1e9, 3), "unit": "GCUPS",
                            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "in_flight": n_fl,
                            "ms_per_step": round(q_ms / e_steps, 3),
                            "note": "xd.Pipeline: the host-API call (H2D of pool + pairs, kernels, D2H) with "
                                    f"{n_fl} batches in flight (one context + host thread each)"}

    # the oracle, as it stands, on a bounded sample (cpu_baseline) -- and the timed batch's results
    # checked against it pair by pair (parity of the number this line reports)
    cpu = None
    parity = None
    chk_w = w.subset(sidx) if n_my != w.n_pairs else w
    if args.scaling == "strong" and world > 1:
        # results of the whole global batch on every rank (untimed): rank 0's parity check below
        # then covers pairs of every shard
        out_d, cells_d = gather_results(out_d, cells_d, sidx, w.n_pairs, world, dev)
        chk_w = w
    if rank == 0 and not args.no_cpu:
        base, (idx, ref, rcells) = oracle_sample(chk_w, args.cpu_seconds if world == 1 else 2.0)
        if world == 1:
            cpu = {k: x for k, x in base.items() if k not in ("sample_s", "sample_pairs")}
        o = out_d.cpu().numpy()[idx]
        c = cells_d.cpu().numpy()[idx]
        bad = np.zeros(idx.shape[0], dtype=bool)
        for i, f in enumerate(("score", "a_begin", "a_end", "b_begin", "b_end")):
            bad |= o[:, i] != ref[f]
        bad |= c != rcells
        parity = {"checked": int(idx.shape[0]), "mismatches": int(bad.sum()),
                  "fields": "score, a_begin, a_end, b_begin, b_end, cells (bit-exact)",
                  "sample": "the cpu_baseline oracle sample (evenly spaced pairs of the timed batch)"}
        if bad.any():
            print(f"PARITY FAILURE: {int(bad.sum())} of {idx.shape[0]} sampled pairs differ from the oracle",
                  file=sys.stderr)

    # the SeqAn/LOGAN-style compat mode (XDROP_FLAG_SEQAN_COMPAT, Q28-Q30) on the same
    # HBM-resident batch: device-timed like `value` (its own cell count), checked against the oracle's
    # compat mode on evenly spaced pairs (informational; not the headline)
    compat = None
    if world == 1 and not args.no_compat:
        with xd.Aligner(devices=[local], seqan_compat=True) as alc:
            oc = torch.zeros_like(out_d)
            cc = torch.zeros_like(cells_d)
            for _ in range(2):
                alc.align_device(seq_d, off_d, pairs_d, oc, cc, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g, stream=stream)
            torch.cuda.synchronize(dev)
            cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
            for a, b in cev:
                flush.zero_()
                a.record(stream)
                alc.align_device(seq_d, off_d, pairs_d, oc, cc, k=w.k, X=w.X, M=w.M, mu=w.mu, g=w.g, stream=stream)
                b.record(stream)
            torch.cuda.synchronize(dev)
            c_ms = min(a.elapsed_time(b) for a, b in cev)
        c_cells = int(cc.sum().item())
        compat = {"value": round(c_cells / (c_ms * 1e-3) / 1e9, 3), "unit": "GCUPS", "ms_per_step": round(c_ms, 3),
                  "cells_per_step": c_cells, "steps": 3, "note": "best of 3 steps, device-resident batch"}
        if rank == 0 and not args.no_cpu:
            import oracle
            idx = np.linspace(0, n_my - 1, min(n_my, 2000)).astype(np.int64)
            ref, rc = oracle.align_batch(w.seq, w.offsets, w.seq, w.offsets, my_pairs[idx], w.k, M=w.M, mu=w.mu,
                                         g=w.g, X=w.X, compat=True)
            o = oc.cpu().numpy()[idx]
            c = cc.cpu().numpy()[idx]
            bad = np.zeros(idx.shape[0], dtype=bool)
            for i, f in enumerate(("score", "a_begin", "a_end", "b_begin", "b_end")):
                bad |= o[:, i] != ref[f]
            bad |= c != rc
            compat["parity"] = {"checked": int(idx.shape[0]), "mismatches": int(bad.sum())}

    if rank == 0:
        line = {"metric": METRIC,
                "value": round(gcups, 3), "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": round(total_ms_max / args.steps, 4),
                "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None,
                "dtype": "i16",
                "per_gpu_ms": [round(x, 3) for x in per_gpu_ms],
                "imbalance": round(max(per_gpu_ms) / (sum(per_gpu_ms) / len(per_gpu_ms)), 4),
                "dtype_note": "DP cell values as packed 16-bit pairs relative to the X-drop threshold; "
                              "scores, thresholds and outputs int32",
                "data": "synthetic", "config": workload_desc(w, args, world),
                "alignments_per_s": round(aps, 1), "cells_per_step": cells_all / args.steps,
                "e2e": e2e, "gpu_launches": int(sum(s["launches"] for s in stats) * world),
                "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "clocks": clocks,
                "escalated_per_step": stats[-1]["escalated"][:3],
                "level_ms": [round(float(x), 3) for x in lvl_ms], "step_ms_all": [round(x, 3) for x in step_ms],
                "compat": compat}
        emit(line, args)
    al.close()


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_native(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
