#!/bin/bash
# round 2, call q (4 GPUs): merged k_hier with 3 and 4 visits per launch; C4 benches
cd $GRAFT_REPO_ROOT
T4="timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29990
for v in 3 4 2; do
port=$((port+1)); MICS_HIER_VISITS=$v $T4 --master-port $port bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2q_c4_n4_v$v.log 2>&1
port=$((port+1)); MICS_HIER_VISITS=$v $T4 --master-port $port bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2q_c4_r4n4_v$v.log 2>&1
done
python tools/show.py gpurun_out/R2q_c*.log | cut -c1-300
