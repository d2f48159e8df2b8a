#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1; tail -2 gpurun_out/u_smoke.log
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29731 bench.py --gpus 4 --sweep > gpurun_out/u_sweep_n4.log 2>&1
python tools/show.py gpurun_out/u_sweep_n4.log | tail -50
