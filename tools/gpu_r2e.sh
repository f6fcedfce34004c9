#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/ab_libs.sh "ecoli xsweep:15 xsweep:50 celegans" paper_2309_07270_b200/libxdrop.so abl/libxdrop_mb4.so > gpurun_out/ab_r2e.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2e.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2e.log
cat gpurun_out/ab_r2e.log; tail -15 gpurun_out/pytest_r2e.log
