#!/bin/bash
cd $GRAFT_REPO_ROOT
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29521 bench.py --gpus 4 --sweep > gpurun_out/sweep_n4.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_n4.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu_n4.log
$T --master-port 29522 bench.py --gpus 4 --ranks 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/b_c3_r4n4.log 2>&1
$T --master-port 29523 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/b_c3_n4.log 2>&1
tail -3 gpurun_out/mgpu_n4.log; grep -c sweep gpurun_out/sweep_n4.log
