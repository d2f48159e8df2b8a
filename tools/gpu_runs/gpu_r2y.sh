#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for f in 0 1; do
MICS_FUSED_BOUNDARY=$f $T2 --master-port 2975$f bench.py --gpus 2 --no-compute --no-e2e > gpurun_out/y_n2_f$f.log 2>&1
MICS_FUSED_BOUNDARY=$f $T4 --master-port 2976$f bench.py --gpus 4 --no-compute --no-e2e > gpurun_out/y_n4_f$f.log 2>&1
MICS_FUSED_BOUNDARY=$f $T4 --master-port 2977$f bench.py --gpus 4 --ranks 4 --no-compute --no-e2e > gpurun_out/y_r4n4_f$f.log 2>&1
MICS_FUSED_BOUNDARY=$f timeout 600 python bench.py --no-compute --no-e2e --no-cpu-baseline > gpurun_out/y_n1_f$f.log 2>&1
done
python tools/show.py gpurun_out/y_*.log
