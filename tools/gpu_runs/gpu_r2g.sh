#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step_compute.py -x -q > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/g_c3_n1.log 2>&1
timeout 600 python bench.py --compute --workload C1 --no-cpu-baseline > gpurun_out/g_c1_cmp_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29652 bench.py --gpus 2 --ranks 2 --compute > gpurun_out/g_c3_cmp_r2n2.log 2>&1
tail -3 gpurun_out/g_tests.log
for f in gpurun_out/g_c*.log; do echo "== $f"; tail -c 3000 $f; echo; done
