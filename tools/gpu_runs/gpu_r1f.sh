#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f_tests.log
tail -3 gpurun_out/f_tests.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/f_c3_n1.log 2>&1
MICS_FUSED_BOUNDARY=0 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/f_c3_n1_unfused.log 2>&1
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29591 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/f_c3_n4.log 2>&1
MICS_FUSED_BOUNDARY=0 $T --master-port 29592 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/f_c3_n4_unfused.log 2>&1
$T --master-port 29593 bench.py --gpus 4 --ranks 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/f_c3_r4n4.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29594 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/f_c3_n2.log 2>&1
