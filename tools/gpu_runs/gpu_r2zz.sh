#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
T4="timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for m in 0 1; do
MICS_HIER_MERGE=$m $T4 --master-port 2995$m bench.py --gpus 4 --workload C4 --steps 3 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/zz_c4_n4_m$m.log 2>&1
MICS_HIER_MERGE=$m $T4 --master-port 2996$m bench.py --gpus 4 --workload C4 --ranks 4 --steps 3 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/zz_c4_r4n4_m$m.log 2>&1
done
python tools/show.py gpurun_out/zz_c4*.log | cut -c1-200
