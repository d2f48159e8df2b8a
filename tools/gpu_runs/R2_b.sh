#!/bin/bash
# round 2, call b (1 GPU): new config-parity + determinism tests, then the whole GPU suite; latency of publish flag
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_determinism.py -q -m gpu > gpurun_out/R2b_new.log 2>&1; echo "rc=$?" >> gpurun_out/R2b_new.log; tail -30 gpurun_out/R2b_new.log
timeout 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_configs.py --deselect tests/test_gpu_determinism.py > gpurun_out/R2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2b_tests.log; tail -3 gpurun_out/R2b_tests.log
