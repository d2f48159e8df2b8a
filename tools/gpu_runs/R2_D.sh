#!/bin/bash
# round 2, call D (4 GPUs): K9 defaults (2 groups, 16 Ki blocks, 2-wave lag) vs the two-kernel boundary:
# C3 N=2, N=4, and one rank per GPU (4 ranks on 4 GPUs, the N=8 shape); parity
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "overlapped_tail or graph_replay" > gpurun_out/R2D_step.log 2>&1; echo "step rc=$?"; tail -2 gpurun_out/R2D_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
port=29850
for rep in 1 2; do
for f in 1 0; do
  port=$((port+1)); MICS_TAIL_FUSED=$f timeout 240 $T --nproc-per-node 2 --master-port $port $B --gpus 2 > gpurun_out/R2D_n2_f${f}_$rep.log 2>&1 || echo "n2 f$f rc=$?"
  port=$((port+1)); MICS_TAIL_FUSED=$f timeout 240 $T --nproc-per-node 4 --master-port $port $B --gpus 4 > gpurun_out/R2D_n4_f${f}_$rep.log 2>&1 || echo "n4 f$f rc=$?"
  port=$((port+1)); MICS_TAIL_FUSED=$f timeout 240 $T --nproc-per-node 4 --master-port $port $B --gpus 4 --ranks 4 > gpurun_out/R2D_r4n4_f${f}_$rep.log 2>&1 || echo "r4n4 f$f rc=$?"
done
done
python tools/show.py gpurun_out/R2D_*.log | cut -c1-200
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2D_mp.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/R2D_mp.log
