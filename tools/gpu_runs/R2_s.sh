#!/bin/bash
# round 2, call s (4 GPUs): final verification — GPU suite, smoke, the driver's bench commands at N=1/2/4,
# the reference arm, C4
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/R2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2s_tests.log; tail -4 gpurun_out/R2s_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/R2s_smoke.log 2>&1; tail -1 gpurun_out/R2s_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/R2s_n1.log 2>&1; echo "n1 rc=$?"
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $T --nproc-per-node 2 --master-port 29711 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/R2s_n2.log 2>&1; echo "n2 rc=$?"
timeout 900 $T --nproc-per-node 4 --master-port 29712 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/R2s_n4.log 2>&1; echo "n4 rc=$?"
timeout 600 $T --nproc-per-node 4 --master-port 29713 bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2s_c4_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29714 bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2s_c4_r4n4.log 2>&1
python tools/show.py gpurun_out/R2s_n*.log gpurun_out/R2s_c4*.log | cut -c1-300
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/R2s_ref_n1.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/R2s_ref_n1.log | cut -c1-300
