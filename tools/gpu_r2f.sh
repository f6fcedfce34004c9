#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/sweep_env.py ecoli "XDROP_KERNEL=0" "XDROP_T0_PER_SM=3" "XDROP_OCC=3" > gpurun_out/sweep_r2f.log 2>&1
timeout 900 python tools/sweep_env.py xsweep:15 "XDROP_KERNEL=0" "XDROP_KERNEL=1" "XDROP_KERNEL=1 XDROP_T0_PER_SM=3" >> gpurun_out/sweep_r2f.log 2>&1
timeout 900 python tools/sweep_env.py celegans "XDROP_KERNEL=0" "XDROP_KERNEL=1" >> gpurun_out/sweep_r2f.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2f.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2f.log
cat gpurun_out/sweep_r2f.log; tail -5 gpurun_out/pytest_r2f.log
