#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/m_tests.log; tail -2 gpurun_out/m_tests.log
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29641 tools/latency.py 2>&1 | grep '^{'
MICS_PDL=0 $T2 --master-port 29643 tools/latency.py 2>&1 | grep '^{'
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/m_n1.log 2>&1
$T2 --master-port 29644 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/m_n2.log 2>&1
$T2 --master-port 29645 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --ranks 2 > gpurun_out/m_r2n2.log 2>&1
for f in gpurun_out/m_n1.log gpurun_out/m_n2.log gpurun_out/m_r2n2.log; do grep -o '"ms_per_step": [0-9.]*\|"phases_ms": {[^}]*}' $f | tr '\n' ' '; echo; done
