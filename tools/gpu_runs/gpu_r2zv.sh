#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k "world" 2>&1 | tail -2
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for d in 0 1; do
MICS_ADAM_DEDUP=$d $T2 --master-port 2996$d bench.py --gpus 2 --no-compute --no-e2e --no-collectives > gpurun_out/zv_n2_d$d.log 2>&1
done
python tools/show.py gpurun_out/zv_n2_*.log | cut -c1-230
