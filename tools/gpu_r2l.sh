#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/sweep_env.py xsweep:15 "XDROP_KERNEL=0" "XDROP_LONG_G=2" "XDROP_LONG_G=2 XDROP_LONG_ALPHA=1" "XDROP_LONG_G=2 XDROP_LONG_ALPHA=4" "XDROP_LONG_G=0" "XDROP_AGE_US=2" > gpurun_out/sweep_r2l.log 2>&1
timeout 900 python tools/sweep_env.py celegans "XDROP_KERNEL=0" "XDROP_LONG_G=2" "XDROP_AGE_US=2" >> gpurun_out/sweep_r2l.log 2>&1
timeout 900 python tools/sweep_env.py ecoli "XDROP_KERNEL=0" "XDROP_LONG_G=2" >> gpurun_out/sweep_r2l.log 2>&1
cat gpurun_out/sweep_r2l.log
