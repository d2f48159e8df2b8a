#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for f in 0 1; do MICS_FUSED_TAIL=$f timeout 600 python bench.py --no-compute --no-e2e --no-cpu-baseline > gpurun_out/zo_n1_f$f.log 2>&1; done
for f in 0 1; do MICS_FUSED_TAIL=$f timeout 600 python bench.py --workload C1 --steps 20 --no-compute --no-e2e --no-cpu-baseline > gpurun_out/zo_c1_f$f.log 2>&1; done
python tools/show.py gpurun_out/zo_*.log | cut -c1-260
