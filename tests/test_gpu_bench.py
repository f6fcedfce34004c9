"""bench.py's contract on a GPU (small config): one JSON line with the driver's keys, measured
roofline peaks, a parity check of the timed batch against the oracle with no mismatch, e2e (per-call
and registered-pool), clocks and launch counts."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_small_config():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "cfg1", "--steps", "3",
                        "--warmup", "3", "--no-traffic", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks",
              "parity", "per_gpu_ms", "imbalance"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "GCUPS" and d["steps"] == 3 and d["warmup"] >= 3
    assert d["parity"]["checked"] == 200 and d["parity"]["mismatches"] == 0
    rf = d["roofline"]
    assert rf["bound"] == "alu" and 0 < rf["frac"] < 1 and rf["peak"] > 1e4      # Gop/s, measured
    assert rf["probes"]["VIMNMX3.S16x2"]["inst_per_clk_sm"] > 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["pooled"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
