#!/bin/bash
cd $GRAFT_REPO_ROOT
MICS_GEMM_PROBE=1 timeout 300 python tools/gemm_bench.py > gpurun_out/v_probe.log 2>&1
grep "gemm probe" gpurun_out/v_probe.log | awk 'NR%23==5'
timeout 300 python tools/gemm_bench.py 2>&1 | cut -c1-200
