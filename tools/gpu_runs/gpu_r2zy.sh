#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for g in 8 12 16; do
MICS_TAIL_GROUPS=$g $T4 --master-port 2997$((g % 10)) bench.py --gpus 4 --no-compute --no-e2e --no-collectives > gpurun_out/zy_n4_g$g.log 2>&1
MICS_TAIL_GROUPS=$g $T2 --master-port 2998$((g % 10)) bench.py --gpus 2 --no-compute --no-e2e --no-collectives > gpurun_out/zy_n2_g$g.log 2>&1
MICS_TAIL_GROUPS=$g $T4 --master-port 2999$((g % 10)) bench.py --gpus 4 --ranks 4 --no-compute --no-e2e --no-collectives > gpurun_out/zy_r4n4_g$g.log 2>&1
done
python tools/show.py gpurun_out/zy_*.log | cut -c1-120
