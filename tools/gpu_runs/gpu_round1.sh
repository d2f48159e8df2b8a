#!/bin/bash
# one gpurun call: multi-GPU parity, NVLink bench (1 rank per GPU) + NCCL comparator, ncu launch list + full capture
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_n2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_n2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --ranks 2 --steps 5 --warmup 3 > gpurun_out/b_c3_r2n2.log 2>&1
CMD="python bench.py --workload C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 8 -c 1 -o gpurun_out/prof_reduce $CMD > gpurun_out/ncu_full.log 2>&1
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_copy -s 40 -c 1 -o gpurun_out/prof_copy $CMD > gpurun_out/ncu_full_copy.log 2>&1
ls -la gpurun_out
