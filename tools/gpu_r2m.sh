#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/sweep_env.py xsweep:15 "XDROP_KERNEL=0" "XDROP_T0_PER_SM=2" "XDROP_T0_PER_SM=2 XDROP_AGE_US=2" "XDROP_T0_PER_SM=2 XDROP_IDLE_NS=2000" > gpurun_out/sweep_r2m.log 2>&1
timeout 900 python tools/sweep_env.py celegans "XDROP_KERNEL=0" "XDROP_T0_PER_SM=2" >> gpurun_out/sweep_r2m.log 2>&1
timeout 900 python tools/sweep_env.py xsweep:50 "XDROP_KERNEL=0" "XDROP_T0_PER_SM=2" >> gpurun_out/sweep_r2m.log 2>&1
timeout 900 python tools/sweep_env.py xsweep:100 "XDROP_KERNEL=0" "XDROP_T0_PER_SM=2" >> gpurun_out/sweep_r2m.log 2>&1
XDROP_T0_PER_SM=2 timeout 300 python tools/timeline.py xsweep:15 > gpurun_out/timeline_xs15_t02.log 2>&1
cat gpurun_out/sweep_r2m.log gpurun_out/timeline_xs15_t02.log
