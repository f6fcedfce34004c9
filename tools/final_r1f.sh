#!/bin/bash
# r1f evidence (run under gpurun; 1 GPU): GPU tests, smoke, bench line, reference arm, ncu launch list
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r1f.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r1f.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r1f.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1f.json 2> gpurun_out/bench_ref_r1f.err; echo "ref rc=$?"
CMD="python bench.py --no-cpu --no-e2e --steps 1 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv $CMD > gpurun_out/ncu_launch_r1f.log 2>&1; echo "launch list rc=$?"
tail -c 2500 gpurun_out/bench_r1f.json; tail -c 1500 gpurun_out/bench_ref_r1f.json; tail -3 gpurun_out/gpu_tests_r1f.log
