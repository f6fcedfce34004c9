#!/bin/bash
# compute-sanitizer over every kernel path (run under gpurun; 1 GPU). Each tool bounded by timeout.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 600 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_run.py --quick > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"
timeout 600 $CS --tool initcheck --error-exitcode 9 python tools/sanitize_run.py --quick > gpurun_out/san_initcheck.log 2>&1; echo "initcheck rc=$?"
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_run.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"
for f in gpurun_out/san_*.log; do echo "== $f"; tail -6 $f; done
