#!/bin/bash
# graph replay + overlapped e2e: tests, A/B at N=1 (C3, C1) and 2 GPUs 1 rank each
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b_tests.log
for g in 0 1; do
  MICS_GRAPH=$g timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_c3_n1_g$g.log 2>&1
  MICS_GRAPH=$g timeout 600 python bench.py --workload C1 --no-cpu-baseline --steps 20 > gpurun_out/b_c1_n1_g$g.log 2>&1
  T2="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
  MICS_GRAPH=$g $T2 --master-port 2962$g bench.py --gpus 2 --ranks 2 > gpurun_out/b_c3_r2n2_g$g.log 2>&1
  MICS_GRAPH=$g $T2 --master-port 2964$g bench.py --gpus 2 --ranks 2 --workload C1 --steps 20 > gpurun_out/b_c1_r2n2_g$g.log 2>&1
done
python tools/show.py gpurun_out/b_*.log
tail -3 gpurun_out/b_tests.log
