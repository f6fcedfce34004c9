#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/ab_libs.sh "xsweep:15 xsweep:50 xsweep:100 celegans ecoli" paper_2309_07270_b200/libxdrop.so abl/libxdrop_cap.so > gpurun_out/ab_r2j.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2j.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_r2j.log
cat gpurun_out/ab_r2j.log; tail -5 gpurun_out/pytest_r2j.log
