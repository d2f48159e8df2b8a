#!/bin/bash
# round 2, call c (4 GPUs): one-launch hierarchical all-gather (k_hier): GPU suite incl. 2/4-GPU
# workers, C4 step n=8 (2 ranks/GPU) and n=4 (1 rank/GPU), C3 N=4 regression
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/R2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2c_tests.log; tail -25 gpurun_out/R2c_tests.log
T4="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29951 bench.py --gpus 4 --workload C4 --steps 5 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2c_c4_n4.log 2>&1
$T4 --master-port 29952 bench.py --gpus 4 --workload C4 --ranks 4 --steps 5 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2c_c4_r4n4.log 2>&1
$T4 --master-port 29953 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2c_c3_n4.log 2>&1
python tools/show.py gpurun_out/R2c_c*.log | cut -c1-300
