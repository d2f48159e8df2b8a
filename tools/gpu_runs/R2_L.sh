#!/bin/bash
# round 2, call L (1 B200): the GPU suite and smoke as the driver runs them on a one-GPU box
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/R2L_tests_1gpu.log 2>&1; echo "rc=$?" >> gpurun_out/R2L_tests_1gpu.log; tail -4 gpurun_out/R2L_tests_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/R2L_smoke.log 2>&1; tail -1 gpurun_out/R2L_smoke.log
