#!/bin/bash
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/zd_trace*
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
MICS_GRAPH=0 MICS_TRACE=gpurun_out/zd_trace.csv $T2 --master-port 29831 bench.py --gpus 2 --ranks 2 --compute --no-e2e --compute-steps 2 > gpurun_out/zd.log 2>&1
python tools/trace_report.py gpurun_out/zd_trace.csv.0 0
