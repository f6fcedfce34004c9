"""Summarise an ncu launch list + one `--set full` capture into profiles/ (run here, no GPU).

usage: python tools/summarize_ncu.py <launches.csv> <prof.ncu-rep> <round-tag>
writes profiles/<tag>_launches.md, profiles/<tag>_band_kernel.md and profiles/ncu_band_kernel.json
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEP_KERNELS = ("pk_tiered_kernel", "pk_merged_kernel", "pk_probe_kernel", "pk_resume_kernel", "band_cta_kernel", "band_merged_kernel", "band_kernel", "general_kernel", "pack_kernel", "prep_kernel",
                "scan_kernel", "scatter_kernel", "combine_kernel", "init_bad_kernel", "init_counters_kernel")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = {}
    for r in data:
        name = r[ki]
        if not any(k in name for k in STEP_KERNELS):
            continue
        per.setdefault(name.split("(")[0], []).append(float(r[vi].replace(",", "")) / 1e6)  # ns -> ms
    return per


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    lpath, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    per = launches(lpath)
    tot = sum(sum(v) for v in per.values())
    lines = [f"# {tag}: ncu launch list of `python bench.py --no-cpu --no-e2e --steps 1 --warmup 3`",
             "", "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares).",
             "Only the kernels of the hot-path step are listed (bench's int32 probe excluded).", "",
             "| kernel | launches | total ms | mean ms | share of step kernels |", "|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.3f} | {sum(v)/len(v):.3f} | {sum(v)/tot:.4f} |")
    open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")

    m = raw_metrics(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
    stall = sorted([(h, v) for h, v in m.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")],
                   key=lambda kv: -float(kv[1][0] or 0))[:8]
    kname = m.get("Kernel Name", ("?", ""))[0]
    md = [f"# {tag}: `ncu --set full` of the dominant kernel", "", f"kernel: `{kname}`", "",
          "| metric | value | unit |", "|---|---|---|"]
    for k in keys:
        if k in m:
            md.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    md += ["", "Top stall reasons (warps per issue-active cycle):", "", "| reason | value |", "|---|---|"]
    for h, v in stall:
        md.append(f"| {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {v[0]} |")
    open(os.path.join(ROOT, "profiles", f"{tag}_band_kernel.md"), "w").write("\n".join(md) + "\n")

    def num(k, scale):
        v, u = m[k]
        v = float(v.replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(u, 1)
        return v * mult / scale
    j = {"tag": tag, "kernel": kname,
         "dram_bytes_per_launch": num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1),
         "duration_ms_under_ncu": num("gpu__time_duration.sum", 1),
         "alu_pipe_pct": float(m["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0]),
         "issue_active_pct": float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
         "registers": int(float(m["launch__registers_per_thread"][0])),
         "source": f"profiles/{tag}_band_kernel.md"}
    json.dump(j, open(os.path.join(ROOT, "profiles", "ncu_band_kernel.json"), "w"), indent=1)
    print("\n".join(lines)); print("\n".join(md)); print(j)


if __name__ == "__main__":
    main()
