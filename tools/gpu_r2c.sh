#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/timeline.py ecoli 20 > gpurun_out/timeline_ecoli.log 2>&1
timeout 600 python tools/sweep_env.py ecoli "XDROP_KERNEL=1" "XDROP_KERNEL=1 XDROP_LONG_G=0" "XDROP_KERNEL=1 XDROP_LONG_ALPHA=2" "XDROP_KERNEL=1 XDROP_STEAL_MIN=0" "XDROP_KERNEL=1 XDROP_STEAL_DIV=4" "XDROP_KERNEL=1 XDROP_T0_PER_SM=2" > gpurun_out/sweep_r2c.log 2>&1
cat gpurun_out/timeline_ecoli.log gpurun_out/sweep_r2c.log
