#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/zf.log 2>&1; echo "rc=$?" >> gpurun_out/zf.log; tail -25 gpurun_out/zf.log
