#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/n_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/n_mgpu.log
tail -30 gpurun_out/n_mgpu.log
