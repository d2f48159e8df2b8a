#!/bin/bash
# round 2, call d (4 GPUs): pipelined hierarchical gathers (k_hier_pipe) vs per-visit k_hier; GPU suite
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/R2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2d_tests.log; tail -25 gpurun_out/R2d_tests.log
T4="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for pipe in 1 0; do
MICS_HIER_PIPE=$pipe $T4 --master-port 2995$pipe bench.py --gpus 4 --workload C4 --steps 5 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2d_c4_n4_p$pipe.log 2>&1
MICS_HIER_PIPE=$pipe $T4 --master-port 2996$pipe bench.py --gpus 4 --workload C4 --ranks 4 --steps 5 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2d_c4_r4n4_p$pipe.log 2>&1
done
python tools/show.py gpurun_out/R2d_c*.log | cut -c1-300
