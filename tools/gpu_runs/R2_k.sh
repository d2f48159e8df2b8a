#!/bin/bash
# round 2, call k (4 GPUs): merged k_hier launches (lag-1 flags, 4 slots): stress, C4 benches, GPU suite, k_hier NVLink
cd $GRAFT_REPO_ROOT
T4="timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for rep in 1 2; do
for m in 1 0; do
MICS_HIER_MERGE=$m $T4 --master-port 2995$m$rep bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2k_c4_n4_m${m}_$rep.log 2>&1
MICS_HIER_MERGE=$m $T4 --master-port 2996$m$rep bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2k_c4_r4n4_m${m}_$rep.log 2>&1
done
done
python tools/show.py gpurun_out/R2k_c*.log | cut -c1-300
timeout 120 python tools/ncu_hier.py > gpurun_out/R2k_hier.log 2>&1; tail -2 gpurun_out/R2k_hier.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/R2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2k_tests.log; tail -4 gpurun_out/R2k_tests.log
