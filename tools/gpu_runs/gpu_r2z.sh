#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29781 bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/z_r2n2_cmp.log 2>&1
tail -c 1500 gpurun_out/z_r2n2_cmp.log
