#!/bin/bash
# gather-slot contents (layers 0-2) after full PDL chains: step tests, full-size C3, multi-GPU
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_multigpu.py -q -m gpu > gpurun_out/r3g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tests.log; tail -3 gpurun_out/r3g_tests.log
