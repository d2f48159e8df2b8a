#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e_tests.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/e_c3_n1.log 2>&1
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --schedule alternative > gpurun_out/e_c3_n1_alt.log 2>&1
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29571 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/e_c3_n2.log 2>&1
$T --master-port 29572 bench.py --gpus 2 --steps 3 --warmup 2 --no-e2e --schedule alternative > gpurun_out/e_c3_n2_alt.log 2>&1
$T --master-port 29573 bench.py --gpus 2 --ranks 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/e_c3_r2n2.log 2>&1
tail -3 gpurun_out/e_tests.log
