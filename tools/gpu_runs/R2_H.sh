#!/bin/bash
# round 2, call H (4 B200): final verification after K9 — GPU suite, smoke, the driver's bench commands at
# N=1/2/4, the reference arm, C4 (n=8 and one rank per GPU), the one-process multi-device bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/R2H_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2H_tests.log; tail -4 gpurun_out/R2H_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/R2H_smoke.log 2>&1; tail -1 gpurun_out/R2H_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/R2H_n1.log 2>&1; echo "n1 rc=$?"
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $T --nproc-per-node 2 --master-port 29961 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/R2H_n2.log 2>&1; echo "n2 rc=$?"
timeout 900 $T --nproc-per-node 4 --master-port 29962 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/R2H_n4.log 2>&1; echo "n4 rc=$?"
timeout 600 $T --nproc-per-node 4 --master-port 29963 bench.py --gpus 4 --workload C4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2H_c4_n4.log 2>&1
timeout 600 $T --nproc-per-node 4 --master-port 29964 bench.py --gpus 4 --workload C4 --ranks 4 --steps 10 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2H_c4_r4n4.log 2>&1
timeout 300 python tools/one_process_bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/R2H_one_process.log 2>&1; tail -1 gpurun_out/R2H_one_process.log | cut -c1-300
python tools/show.py gpurun_out/R2H_n*.log gpurun_out/R2H_c4*.log | cut -c1-300
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/R2H_ref_n1.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/R2H_ref_n1.log | cut -c1-300
