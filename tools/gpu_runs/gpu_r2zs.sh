#!/bin/bash
cd $GRAFT_REPO_ROOT
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for t in 0 1; do
MICS_TAIL_OVERLAP=$t $T4 --master-port 2992$t bench.py --gpus 4 --ranks 4 --no-compute --no-e2e --no-collectives > gpurun_out/zs_r4n4_t$t.log 2>&1
MICS_TAIL_OVERLAP=$t $T4 --master-port 2993$t bench.py --gpus 4 --ranks 4 --p 4 --no-compute --no-e2e --no-collectives > gpurun_out/zs_r4n4p4_t$t.log 2>&1
done
python tools/show.py gpurun_out/zs_*.log | cut -c1-230
