#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l_tests.log; tail -2 gpurun_out/l_tests.log
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29641 tools/latency.py 2>&1 | grep '^{'
MICS_BAR_STRICT=1 $T2 --master-port 29642 tools/latency.py 2>&1 | grep '^{'
MICS_PDL=0 $T2 --master-port 29643 tools/latency.py 2>&1 | grep '^{'
for i in 1 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2965$i tests/mp_worker.py > gpurun_out/l_mp$i.log 2>&1; echo "mp rc=$?"; done
$T2 --master-port 29644 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --ranks 2 > gpurun_out/l_r2n2.log 2>&1
grep -o '"ms_per_step": [0-9.]*\|"phases_ms": {[^}]*}' gpurun_out/l_r2n2.log
