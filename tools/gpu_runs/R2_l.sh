#!/bin/bash
# round 2, call l (4 GPUs): C4 benches, merged k_hier launches vs one per visit, twice
cd $GRAFT_REPO_ROOT
T4="timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29960
for rep in 1 2; do
for m in 1 0; do
port=$((port+1)); MICS_HIER_MERGE=$m $T4 --master-port $port bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2l_c4_n4_m${m}_$rep.log 2>&1
port=$((port+1)); MICS_HIER_MERGE=$m $T4 --master-port $port bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2l_c4_r4n4_m${m}_$rep.log 2>&1
done
done
python tools/show.py gpurun_out/R2l_c*.log | cut -c1-300
