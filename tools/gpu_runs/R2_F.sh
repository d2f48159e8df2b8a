#!/bin/bash
# round 2, call F (4 GPUs): K10 (last reduce-scatter + boundary + Adam in one k_fbnd launch) — parity on one GPU
# (forced) and across 2/4 GPU processes, then C3 N=2/N=4, one rank per GPU, and C4 against K9
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "fused_tail or overlapped_tail or graph_replay" > gpurun_out/R2F_step.log 2>&1; echo "step rc=$?"; tail -2 gpurun_out/R2F_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
timeout 240 $T --nproc-per-node 2 --master-port 29901 $B --gpus 2 > gpurun_out/R2F_n2_k10.log 2>&1; rc=$?; echo "first rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2F_mp.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/R2F_mp.log
port=29910
for v in k10 k9; do
  if [ $v = k9 ]; then E="MICS_FTAIL=0"; else E="MICS_FTAIL=1"; fi
  port=$((port+1)); env $E timeout 240 $T --nproc-per-node 2 --master-port $port $B --gpus 2 > gpurun_out/R2F_n2_$v.log 2>&1 || echo "n2 $v rc=$?"
  port=$((port+1)); env $E timeout 240 $T --nproc-per-node 4 --master-port $port $B --gpus 4 > gpurun_out/R2F_n4_$v.log 2>&1 || echo "n4 $v rc=$?"
  port=$((port+1)); env $E timeout 240 $T --nproc-per-node 4 --master-port $port $B --gpus 4 --ranks 4 > gpurun_out/R2F_r4n4_$v.log 2>&1 || echo "r4n4 $v rc=$?"
  port=$((port+1)); env $E timeout 400 $T --nproc-per-node 4 --master-port $port bench.py --workload C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-compute --no-collectives --gpus 4 > gpurun_out/R2F_c4_$v.log 2>&1 || echo "c4 $v rc=$?"
done
python tools/show.py gpurun_out/R2F_*.log | cut -c1-220
