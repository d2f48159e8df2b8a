#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d_tests.log
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29561 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/d_c3_n4.log 2>&1
$T --master-port 29562 bench.py --gpus 4 --ranks 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/d_c3_r4n4.log 2>&1
$T --master-port 29563 bench.py --gpus 4 --workload C4 --ranks 4 --steps 3 --warmup 2 --no-e2e > gpurun_out/d_c4_r4n4.log 2>&1
$T --master-port 29564 bench.py --gpus 4 --workload C5p8 --steps 2 --warmup 2 --no-e2e > gpurun_out/d_c5p8_n4.log 2>&1
CMD="python bench.py --workload C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 5 -c 4 -o gpurun_out/prof_reduce_v2 $CMD > gpurun_out/d_ncu.log 2>&1
$CMD > gpurun_out/d_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_v2.csv $CMD > gpurun_out/d_ncu_list.log 2>&1
tail -2 gpurun_out/d_tests.log
