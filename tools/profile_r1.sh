#!/bin/bash
# ncu evidence for the bench's dominant kernel (run under gpurun; 1 GPU)
set -u
mkdir -p gpurun_out
CMD="python bench.py --no-cpu --no-e2e --steps 1 --warmup 3"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:band_merged -s 3 -c 1 -o gpurun_out/prof_r1d $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
