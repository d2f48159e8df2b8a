#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/d_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/d_gemm.log
tail -30 gpurun_out/d_gemm.log
