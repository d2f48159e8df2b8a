#!/bin/bash
# quick check on 2 GPUs: gpu tests, N=1 bench, p=2 sweep, 2-rank NVLink bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_b_n1.log 2>&1
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29541 bench.py --gpus 2 --sweep > gpurun_out/q_sweep_n2.log 2>&1
$T --master-port 29542 bench.py --gpus 2 --ranks 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/q_b_r2n2.log 2>&1
tail -2 gpurun_out/q_tests.log
