#!/bin/bash
# round 2, call N (2 B200): after the K9 descriptor clean-up — K9 parity on one GPU, across processes, the flag stress
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_barrier_stress.py tests/test_gpu_fullsize.py tests/test_multigpu.py -q > gpurun_out/R2N_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/R2N_tests.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 2 --master-port 29995 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives > gpurun_out/R2N_n2.log 2>&1; echo "n2 rc=$?"
python tools/show.py gpurun_out/R2N_n2.log | cut -c1-200
