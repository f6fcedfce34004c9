#!/bin/bash
# round-2 evidence run: GPU tests, configs 1-5 throughput, config 5 at full scale (5M pairs), bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r2n.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2n.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2n.log
timeout 1200 python tools/configs_bench.py --out gpurun_out/configs_r2n.md > gpurun_out/configs_r2n.log 2>&1
timeout 1500 python tools/celegans_full.py --out gpurun_out/celegans_full_r2n.md > gpurun_out/celegans_full_r2n.log 2>&1
timeout 900 python bench.py --out gpurun_out/bench_r2n.json > gpurun_out/bench_r2n.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench_r2n.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --out gpurun_out/bench_ref_r2n.json > gpurun_out/bench_ref_r2n.log 2>&1
tail -3 gpurun_out/pytest_r2n.log; cat gpurun_out/configs_r2n.md; cat gpurun_out/celegans_full_r2n.md; tail -c 600 gpurun_out/bench_r2n.log; tail -c 400 gpurun_out/bench_ref_r2n.log
