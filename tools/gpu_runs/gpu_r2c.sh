#!/bin/bash
# 8-GPU: default bench (the driver's scaling point) + C2 sweep at p=2/4/8
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/c_topo.log 2>&1
T8="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
$T8 --master-port 29711 bench.py --gpus 8 > gpurun_out/c_n8.log 2>&1
$T8 --master-port 29712 bench.py --gpus 8 --sweep > gpurun_out/c_sweep_n8.log 2>&1
python tools/show.py gpurun_out/c_n8.log gpurun_out/c_sweep_n8.log
