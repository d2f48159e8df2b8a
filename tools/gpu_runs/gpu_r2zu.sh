#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_gpu_step.py -x -q > gpurun_out/zu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zu_tests.log; tail -3 gpurun_out/zu_tests.log
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29951 bench.py --gpus 4 --workload C4 --steps 3 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/zu_c4_n4.log 2>&1
$T4 --master-port 29952 bench.py --gpus 4 --workload C4 --ranks 4 --steps 3 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/zu_c4_r4n4.log 2>&1
python tools/show.py gpurun_out/zu_c4*.log | cut -c1-260
