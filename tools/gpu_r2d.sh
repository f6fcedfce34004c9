#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2d.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2d.log
timeout 600 python tools/sweep_env.py xsweep:15 "XDROP_KERNEL=0" > gpurun_out/sweep_r2d.log 2>&1
timeout 600 python tools/sweep_env.py celegans "XDROP_KERNEL=0" >> gpurun_out/sweep_r2d.log 2>&1
timeout 600 python tools/sweep_env.py ecoli "XDROP_KERNEL=0" >> gpurun_out/sweep_r2d.log 2>&1
timeout 900 python tools/celegans_full.py > gpurun_out/celegans_full_r2d.log 2>&1
tail -3 gpurun_out/pytest_r2d.log; cat gpurun_out/sweep_r2d.log; tail -20 gpurun_out/celegans_full_r2d.log
