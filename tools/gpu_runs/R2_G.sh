#!/bin/bash
# round 2, call G (4 GPUs): K10 with an unrolled stage A and K9 back at 4 Adam rows; N=1 forced K10 vs K8
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "fused_tail or overlapped_tail or graph_replay" > gpurun_out/R2G_step.log 2>&1; echo "step rc=$?"; tail -2 gpurun_out/R2G_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
timeout 300 python $B > gpurun_out/R2G_n1_k8.log 2>&1 || echo "n1 k8 rc=$?"
MICS_FTAIL=2 MICS_FUSED_TAIL=0 timeout 300 python $B > gpurun_out/R2G_n1_k10.log 2>&1 || echo "n1 k10 rc=$?"
port=29930
for v in k10 k9; do
  if [ $v = k9 ]; then E="MICS_FTAIL=0"; else E="MICS_FTAIL=1"; fi
  port=$((port+1)); env $E timeout 240 $T --nproc-per-node 2 --master-port $port $B --gpus 2 > gpurun_out/R2G_n2_$v.log 2>&1 || echo "n2 $v rc=$?"
  port=$((port+1)); env $E timeout 240 $T --nproc-per-node 4 --master-port $port $B --gpus 4 > gpurun_out/R2G_n4_$v.log 2>&1 || echo "n4 $v rc=$?"
done
python tools/show.py gpurun_out/R2G_*.log | cut -c1-220
