#!/bin/bash
# round 2, call j (4 GPUs): GPU suite after the pipe removal; C4 / C3 benches at 2 and 4 GPUs;
# C2 sweep with the graph-captured NCCL comparator; k_hier NVLink timing (one process, 2 GPUs)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/R2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2j_tests.log; tail -4 gpurun_out/R2j_tests.log
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
T4="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29951 bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2j_c4_n4.log 2>&1
$T4 --master-port 29952 bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2j_c4_r4n4.log 2>&1
$T2 --master-port 29953 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2j_c3_n2.log 2>&1
$T4 --master-port 29954 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2j_c3_n4.log 2>&1
python tools/show.py gpurun_out/R2j_c*.log | cut -c1-300
timeout 120 python tools/ncu_hier.py > gpurun_out/R2j_hier.log 2>&1; cat gpurun_out/R2j_hier.log | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29955 bench.py --gpus 4 --sweep --steps 5 > gpurun_out/R2j_sweep_n4.log 2>&1
python tools/show.py gpurun_out/R2j_sweep_n4.log
