#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/zg.log 2>&1; echo "rc=$?" >> gpurun_out/zg.log; tail -25 gpurun_out/zg.log
