#!/bin/bash
# r1e evidence (run under gpurun; 1 GPU): bench line, ncu launch list + full capture of the bench's
# dominant kernel, a full capture of the shared kernel on C. elegans x0.05, configs table, config 5
set -u
mkdir -p gpurun_out
CMD="python bench.py --no-cpu --no-e2e --steps 1 --warmup 3"
python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:pk_tiered -s 3 -c 1 -o gpurun_out/prof_r1e $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:pk_merged -s 0 -c 1 -o gpurun_out/prof_r1e_cel python tools/run_cfg.py celegans 2 > gpurun_out/ncu_cel.log 2>&1; echo "cel rc=$?"
python tools/configs_bench.py --out gpurun_out/configs_r1.md > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
python tools/celegans_full.py --scale 1.0 --out gpurun_out/celegans_full_r1.md > gpurun_out/celfull.log 2>&1; echo "celfull rc=$?"
