#!/bin/bash
# re-entry check on 2 GPUs: gpu tests, smoke, default N=1 bench + reference arm, N=2 bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/a_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/a_n1.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/a_ref_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29611 bench.py --gpus 2 > gpurun_out/a_n2.log 2>&1
for f in gpurun_out/a_*.log; do echo "== $f"; tail -c 1200 $f; echo; done
