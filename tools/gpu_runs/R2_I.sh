#!/bin/bash
# round 2, call I (2 B200): full-size C3 every-element checks (1 GPU: K8 and K9; 2 processes: K9), K9 flag stress
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_barrier_stress.py -q > gpurun_out/R2I_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/R2I_tests.log
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2I_mp.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/R2I_mp.log
