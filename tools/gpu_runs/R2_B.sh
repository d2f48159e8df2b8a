#!/bin/bash
# round 2, call B (4 GPUs): K9 rounds with a wave-sized lag; block 64Ki / 16Ki elements; layer groups 8 / 2
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "overlapped_tail or graph_replay" > gpurun_out/R2B_step.log 2>&1; echo "step rc=$?"; tail -2 gpurun_out/R2B_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
MICS_TAIL_FUSED=1 timeout 240 $T --nproc-per-node 2 --master-port 29801 $B --gpus 2 > gpurun_out/R2B_n2_first.log 2>&1; rc=$?; echo "first rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
port=29810
for v in f0g8b64 f1g8b64 f1g8b16 f1g2b64 f1g2b16 f1g4b16; do
  for n in 2 4; do
    port=$((port+1))
    MICS_TAIL_FUSED=${v:1:1} MICS_TAIL_GROUPS=${v:3:1} MICS_FB_BLOCK=$((${v:5:2}*1024)) timeout 240 $T --nproc-per-node $n --master-port $port $B --gpus $n > gpurun_out/R2B_n${n}_$v.log 2>&1 || echo "n$n $v rc=$?"
  done
done
python tools/show.py gpurun_out/R2B_n*.log | cut -c1-260
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2B_mp.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/R2B_mp.log
