#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_gpu_step.py -x -q > gpurun_out/zr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zr_tests.log; tail -3 gpurun_out/zr_tests.log
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for t in 0 1; do
MICS_TAIL_OVERLAP=$t $T2 --master-port 2990$t bench.py --gpus 2 --no-compute --no-e2e --no-collectives > gpurun_out/zr_n2_t$t.log 2>&1
MICS_TAIL_OVERLAP=$t $T4 --master-port 2991$t bench.py --gpus 4 --no-compute --no-e2e --no-collectives > gpurun_out/zr_n4_t$t.log 2>&1
done
python tools/show.py gpurun_out/zr_n*.log | cut -c1-230
