#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S=gpurun_out/sweep_r2b.log
timeout 600 python tools/sweep_env.py xsweep:15 "XDROP_KERNEL=1" "XDROP_KERNEL=2" "XDROP_KERNEL=1 XDROP_LONG_G=0" "XDROP_KERNEL=2 XDROP_LONG_G=0" "XDROP_KERNEL=1 XDROP_LONG_ALPHA=4" "XDROP_KERNEL=1 XDROP_LONG_ALPHA=0.3" "XDROP_KERNEL=1 XDROP_OCC=2" "XDROP_KERNEL=1 XDROP_OCC=1" "XDROP_KERNEL=1 XDROP_LONG_G=2" > $S 2>&1
timeout 600 python tools/sweep_env.py celegans "XDROP_KERNEL=1" "XDROP_KERNEL=2" "XDROP_KERNEL=2 XDROP_LONG_G=0" "XDROP_KERNEL=2 XDROP_OCC=2" "XDROP_KERNEL=1 XDROP_LONG_G=0" >> $S 2>&1
timeout 300 python tools/timeline.py xsweep:15 > gpurun_out/timeline_xs15.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pk_tiered_kernel -s 2 -c 1 -o gpurun_out/r2b_ecoli python tools/run_cfg.py ecoli 3 > gpurun_out/ncu_r2b.log 2>&1
tail -30 $S; tail -30 gpurun_out/timeline_xs15.log; tail -3 gpurun_out/ncu_r2b.log
