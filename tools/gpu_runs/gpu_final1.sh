#!/bin/bash
# the driver's round-end invocations (default flags)
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/z_n1.log 2>&1
python bench.py --impl reference > gpurun_out/z_ref_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29611 bench.py --gpus 2 > gpurun_out/z_n2.log 2>&1
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29612 bench.py --gpus 4 > gpurun_out/z_n4.log 2>&1
$T4 --master-port 29613 bench.py --gpus 4 --impl reference > gpurun_out/z_ref_n4.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1
for f in gpurun_out/z_*.log; do echo "== $f"; tail -c 1500 $f; echo; done
