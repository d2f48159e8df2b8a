#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/j_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/j_gemm.log
tail -5 gpurun_out/j_gemm.log
timeout 300 python tools/gemm_bench.py > gpurun_out/j_gemm_bench.log 2>&1; cat gpurun_out/j_gemm_bench.log
