#!/bin/bash
cd $GRAFT_REPO_ROOT
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 1 2 3; do
MICS_COPY_CTAS_PER_SM=$c $T --master-port 2958$c bench.py --gpus 2 --ranks 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/t_ctas$c.log 2>&1
done
MICS_PDL=0 $T --master-port 29589 bench.py --gpus 2 --ranks 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/t_nopdl.log 2>&1
