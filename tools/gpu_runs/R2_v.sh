#!/bin/bash
# round 2, call v (4 GPUs): K9 fused layer-group boundary — parity (1 GPU overlapped tail, multi-process
# overlapped tail at world 2/4) and C3 N=2/N=4 with MICS_TAIL_FUSED=0/1
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step.py -q -k "overlapped_tail or graph_replay" > gpurun_out/R2v_step.log 2>&1; echo "step rc=$?"; tail -3 gpurun_out/R2v_step.log
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2v_mp.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/R2v_mp.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
port=29721
for f in 1 0; do
  for n in 2 4; do
    port=$((port+1))
    MICS_TAIL_FUSED=$f timeout 600 $T --nproc-per-node $n --master-port $port $B --gpus $n > gpurun_out/R2v_n${n}_f$f.log 2>&1; echo "n$n f$f rc=$?"
  done
done
python tools/show.py gpurun_out/R2v_n*.log | cut -c1-400
