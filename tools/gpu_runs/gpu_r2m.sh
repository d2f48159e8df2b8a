#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_bench.py > gpurun_out/m_gemm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 23 -c 1 -o gpurun_out/m_gemm_fwd python tools/gemm_bench.py > gpurun_out/m_ncu_gemm.log 2>&1
timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --compute-steps 2 > gpurun_out/m_cmp_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/m_launches_cmp.csv python bench.py --compute --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --compute-steps 2 > gpurun_out/m_ncu_cmp.log 2>&1
tail -2 gpurun_out/m_ncu_gemm.log gpurun_out/m_ncu_cmp.log; ls -la gpurun_out/m_*
