#!/bin/bash
# round 2, call u (2 GPUs): new multi-device compute test + the GPU suite on 2 GPUs; one-process bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/R2u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2u_tests.log; tail -4 gpurun_out/R2u_tests.log
timeout 300 python tools/one_process_bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/R2u_one_process.log 2>&1; tail -1 gpurun_out/R2u_one_process.log
