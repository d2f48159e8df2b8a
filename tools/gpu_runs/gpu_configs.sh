#!/bin/bash
# C4 (hierarchical) and C5 (10B) step configs on 4 GPUs
cd $GRAFT_REPO_ROOT
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29551 bench.py --gpus 4 --workload C4 --steps 3 --warmup 2 --no-e2e > gpurun_out/c_c4_n4.log 2>&1
$T --master-port 29552 bench.py --gpus 4 --workload C4 --ranks 4 --steps 3 --warmup 2 --no-e2e > gpurun_out/c_c4_r4n4.log 2>&1
$T --master-port 29553 bench.py --gpus 4 --workload C5p8 --steps 2 --warmup 2 --no-e2e > gpurun_out/c_c5p8_n4.log 2>&1
$T --master-port 29554 bench.py --gpus 4 --workload C3 --steps 5 --warmup 3 > gpurun_out/c_c3_n4.log 2>&1
python bench.py --workload C4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/c_c4_n1.log 2>&1
for f in gpurun_out/c_*.log; do echo $f; tail -2 $f | cut -c1-300; done
