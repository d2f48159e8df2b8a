#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_step_compute.py -x -q > gpurun_out/w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w_tests.log; tail -3 gpurun_out/w_tests.log
MICS_GEMM_PROBE=1 timeout 300 python tools/gemm_bench.py > gpurun_out/w_probe.log 2>&1
grep "gemm probe" gpurun_out/w_probe.log | awk 'NR%23==5'
timeout 300 python tools/gemm_bench.py 2>&1 | cut -c1-180
MICS_GEMM_TMA_STORE=0 timeout 300 python tools/gemm_bench.py 2>&1 | cut -c1-180
