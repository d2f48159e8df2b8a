#!/bin/bash
# round 2, call A (4 GPUs): K9 with rounds (fold of block t, Adam of block t-2) — parity, then N=2/4 vs the
# two-kernel boundary, layer groups 8 / 4 / 2
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "overlapped_tail or graph_replay" > gpurun_out/R2A_step.log 2>&1; echo "step rc=$?"; tail -2 gpurun_out/R2A_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
MICS_TAIL_FUSED=1 timeout 240 $T --nproc-per-node 2 --master-port 29781 $B --gpus 2 > gpurun_out/R2A_n2_f1g8.log 2>&1; rc=$?; echo "first rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
port=29790
for v in f0g8 f1g8 f1g4 f1g2 f0g4; do
  for n in 2 4; do
    port=$((port+1))
    MICS_TAIL_FUSED=${v:1:1} MICS_TAIL_GROUPS=${v:3:1} timeout 240 $T --nproc-per-node $n --master-port $port $B --gpus $n > gpurun_out/R2A_n${n}_$v.log 2>&1 || echo "n$n $v rc=$?"
  done
done
python tools/show.py gpurun_out/R2A_n*.log | cut -c1-300
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2A_mp.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/R2A_mp.log
