#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2h.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2h.log
timeout 900 python tools/sweep_env.py xsweep:15 "XDROP_KERNEL=0" "XDROP_LONG_ALPHA=2" "XDROP_LONG_ALPHA=4" "XDROP_STEAL_DIV=2" "XDROP_STEAL_DIV=32" > gpurun_out/sweep_r2h.log 2>&1
timeout 900 python tools/sweep_env.py celegans "XDROP_KERNEL=0" "XDROP_LONG_ALPHA=2" "XDROP_LONG_ALPHA=4" >> gpurun_out/sweep_r2h.log 2>&1
timeout 900 python tools/sweep_env.py ecoli "XDROP_KERNEL=0" "XDROP_LONG_ALPHA=2" "XDROP_LONG_ALPHA=4" >> gpurun_out/sweep_r2h.log 2>&1
tail -5 gpurun_out/pytest_r2h.log; cat gpurun_out/sweep_r2h.log
