#!/bin/bash
# round 2, call o (4 GPUs): merged k_hier with done counters: C4 benches (merged vs per visit), hier tests
cd $GRAFT_REPO_ROOT
T4="timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29970
for m in 1 0; do
port=$((port+1)); MICS_HIER_MERGE=$m $T4 --master-port $port bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2o_c4_n4_m$m.log 2>&1
port=$((port+1)); MICS_HIER_MERGE=$m $T4 --master-port $port bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2o_c4_r4n4_m$m.log 2>&1
done
python tools/show.py gpurun_out/R2o_c*.log | cut -c1-300
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_step.py tests/test_multigpu.py tests/test_gpu_configs.py -k "hier or c4 or across" > gpurun_out/R2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2o_tests.log; tail -4 gpurun_out/R2o_tests.log
