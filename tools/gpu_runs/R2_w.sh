#!/bin/bash
# round 2, call w (4 GPUs): K9 after the flag-stride fix — short bench first (bounded), then parity
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "overlapped_tail or graph_replay" > gpurun_out/R2w_step.log 2>&1; echo "step rc=$?"; tail -3 gpurun_out/R2w_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
MICS_TAIL_FUSED=1 timeout 240 $T --nproc-per-node 2 --master-port 29731 $B --gpus 2 > gpurun_out/R2w_n2_f1.log 2>&1; rc=$?; echo "n2 f1 rc=$rc"
if [ $rc -ne 0 ]; then exit 1; fi
MICS_TAIL_FUSED=1 timeout 240 $T --nproc-per-node 4 --master-port 29732 $B --gpus 4 > gpurun_out/R2w_n4_f1.log 2>&1; echo "n4 f1 rc=$?"
MICS_TAIL_FUSED=0 timeout 240 $T --nproc-per-node 2 --master-port 29733 $B --gpus 2 > gpurun_out/R2w_n2_f0.log 2>&1; echo "n2 f0 rc=$?"
MICS_TAIL_FUSED=0 timeout 240 $T --nproc-per-node 4 --master-port 29734 $B --gpus 4 > gpurun_out/R2w_n4_f0.log 2>&1; echo "n4 f0 rc=$?"
python tools/show.py gpurun_out/R2w_n*.log | cut -c1-400
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/R2w_mp.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/R2w_mp.log
