#!/bin/bash
# round 2, call a (2 GPUs): GPU suite after the prune + exit-barrier fences; latency; N=1/2 bench
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/R2a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2a_tests.log; tail -3 gpurun_out/R2a_tests.log
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29641 tools/latency.py 2>&1 | grep '^{' > gpurun_out/R2a_lat.log
MICS_BAR_STRICT=1 $T2 --master-port 29642 tools/latency.py 2>&1 | grep '^{' >> gpurun_out/R2a_lat.log
cat gpurun_out/R2a_lat.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-compute > gpurun_out/R2a_n1.log 2>&1
$T2 --master-port 29644 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2a_n2.log 2>&1
for f in gpurun_out/R2a_n1.log gpurun_out/R2a_n2.log; do grep -o '"ms_per_step": [0-9.]*\|"phases_ms": {[^}]*}' $f | tr '\n' ' '; echo; done
