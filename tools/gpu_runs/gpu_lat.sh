#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 python tools/latency.py 2>&1 | tail -2
$T2 --master-port 29641 tools/latency.py 2>&1 | grep '^{'
MICS_PDL=0 $T2 --master-port 29642 tools/latency.py 2>&1 | grep '^{'
