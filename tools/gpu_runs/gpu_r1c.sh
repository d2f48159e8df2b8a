#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_n4.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_n4.log
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29531 bench.py --gpus 4 --sweep > gpurun_out/sweep_n4.log 2>&1
$T --master-port 29532 bench.py --gpus 4 --ranks 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/b_c3_r4n4.log 2>&1
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_c3_n1.log 2>&1
tail -3 gpurun_out/gpu_tests_n4.log
