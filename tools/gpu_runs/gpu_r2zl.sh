#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 240 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -4
for pr in 2 1; do echo "== PAIRS=$pr"; MICS_GEMM_PAIRS=$pr timeout 240 python tools/gemm_bench.py 2>&1 | cut -c1-170; done
