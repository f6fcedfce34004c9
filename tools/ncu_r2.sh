#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
./tools/pk_unit > gpurun_out/pk_unit.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2g.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2g.log
timeout 900 python bench.py --out gpurun_out/bench_r2g.json > gpurun_out/bench_r2g.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench_r2g.log
timeout 900 python tools/sweep_env.py ecoli "XDROP_KERNEL=0" "XDROP_OCC=2" "XDROP_LONG_ALPHA=2" "XDROP_LONG_ALPHA=0.5" > gpurun_out/sweep_r2g.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2g.csv python bench.py --steps 2 --warmup 1 --no-traffic --no-cpu --no-e2e > gpurun_out/ncu_launch_r2g.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pk_tiered_kernel -s 3 -c 1 -o gpurun_out/r2g_ecoli python bench.py --steps 1 --warmup 3 --no-traffic --no-cpu --no-e2e > gpurun_out/ncu_full_r2g.log 2>&1
cat gpurun_out/pk_unit.log; tail -3 gpurun_out/pytest_r2g.log; tail -c 1500 gpurun_out/bench_r2g.log; cat gpurun_out/sweep_r2g.log; tail -2 gpurun_out/ncu_full_r2g.log
