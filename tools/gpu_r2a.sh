#!/bin/bash
# round-2 GPU check: full GPU test suite, then the default bench (with its ncu traffic child)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest.log; tail -c 600 gpurun_out/bench.log
