#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
tail -3 gpurun_out/h_tests.log
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29601 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/h_c3_n4.log 2>&1
MICS_PIPELINE=0 $T --master-port 29602 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/h_c3_n4_nopipe.log 2>&1
$T --master-port 29603 bench.py --gpus 4 --ranks 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/h_c3_r4n4.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29604 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/h_c3_n2.log 2>&1
