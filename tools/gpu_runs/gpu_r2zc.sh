#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/zc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zc_tests.log; tail -3 gpurun_out/zc_tests.log
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/zc_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/zc_mgpu.log; tail -3 gpurun_out/zc_mgpu.log
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for t in 0 1; do
MICS_TAIL_OVERLAP=$t $T2 --master-port 2980$t bench.py --gpus 2 --no-compute --no-e2e > gpurun_out/zc_n2_t$t.log 2>&1
MICS_TAIL_OVERLAP=$t $T4 --master-port 2981$t bench.py --gpus 4 --no-compute --no-e2e > gpurun_out/zc_n4_t$t.log 2>&1
MICS_TAIL_OVERLAP=$t $T4 --master-port 2982$t bench.py --gpus 4 --ranks 4 --no-compute --no-e2e > gpurun_out/zc_r4n4_t$t.log 2>&1
MICS_TAIL_OVERLAP=$t timeout 600 python bench.py --no-compute --no-e2e --no-cpu-baseline > gpurun_out/zc_n1_t$t.log 2>&1
done
python tools/show.py gpurun_out/zc_n*.log gpurun_out/zc_r4*.log | cut -c1-250
