#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/timeline.py xsweep:15 > gpurun_out/timeline_xs15_r2k.log 2>&1
TL_KERNEL=1 timeout 300 python tools/timeline.py xsweep:15 > gpurun_out/timeline_xs15t_r2k.log 2>&1
timeout 300 python tools/timeline.py xsweep:50 > gpurun_out/timeline_xs50_r2k.log 2>&1
timeout 300 python tools/timeline.py celegans > gpurun_out/timeline_ce_r2k.log 2>&1
cat gpurun_out/timeline_xs15_r2k.log gpurun_out/timeline_xs15t_r2k.log gpurun_out/timeline_xs50_r2k.log gpurun_out/timeline_ce_r2k.log
