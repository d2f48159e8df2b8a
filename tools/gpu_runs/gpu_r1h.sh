#!/bin/bash
# slice-interleaved Adam tiles: parity + boundary phase at N=4/2/1
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/i_tests.log
tail -3 gpurun_out/i_tests.log
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29601 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/i_c3_n4.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29604 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/i_c3_n2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/i_c3_n1.log 2>&1
for f in gpurun_out/i_c3_*.log; do echo "== $f"; grep -E "phase|boundary|^\{" $f | tail -c 1800; echo; done
