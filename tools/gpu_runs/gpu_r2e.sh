#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_bench.py > gpurun_out/e_gemm.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 12 -c 1 -o gpurun_out/e_gemm_fwd python tools/gemm_bench.py > gpurun_out/e_ncu.log 2>&1
cat gpurun_out/e_gemm.log; tail -3 gpurun_out/e_ncu.log
