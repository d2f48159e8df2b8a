#!/bin/bash
# round 2, call e (2 GPUs): per-launch tickets for k_hier_pipe; multi-device context tests; barrier stress
cd $GRAFT_REPO_ROOT
T2="timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for pipe in 1 0; do
MICS_HIER_PIPE=$pipe $T2 --master-port 2995$pipe bench.py --gpus 2 --workload C4 --ranks 4 --steps 5 --warmup 3 --no-e2e --no-compute --no-collectives > gpurun_out/R2e_c4_r4n2_p$pipe.log 2>&1
done
python tools/show.py gpurun_out/R2e_c*.log | cut -c1-300
timeout 900 python -m pytest -x -q tests/test_gpu_step.py tests/test_gpu_multidevice.py tests/test_gpu_barrier_stress.py tests/test_reference_suites.py tests/test_gpu_parity.py > gpurun_out/R2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2e_tests.log; tail -30 gpurun_out/R2e_tests.log
