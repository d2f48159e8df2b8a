#!/bin/bash
# round 2, call p (4 GPUs): merged k_hier with 1 vs 2 visits per launch; C4 benches; hier tests
cd $GRAFT_REPO_ROOT
T4="timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29980
for v in 2 1; do
port=$((port+1)); MICS_HIER_VISITS=$v $T4 --master-port $port bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2p_c4_n4_v$v.log 2>&1
port=$((port+1)); MICS_HIER_VISITS=$v $T4 --master-port $port bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2p_c4_r4n4_v$v.log 2>&1
done
python tools/show.py gpurun_out/R2p_c*.log | cut -c1-300
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_step.py tests/test_multigpu.py tests/test_gpu_configs.py -k "hier or c4 or across" > gpurun_out/R2p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2p_tests.log; tail -4 gpurun_out/R2p_tests.log
