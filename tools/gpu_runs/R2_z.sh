#!/bin/bash
# round 2, call z (4 GPUs): K9 grid (persistent vs one CTA per item) x tail reduce-scatter priority; compute step N=1
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_step.py -q -k "overlapped_tail or graph_replay" > gpurun_out/R2z_step.log 2>&1; echo "step rc=$?"; tail -2 gpurun_out/R2z_step.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
port=29770
for v in f0 c2p1 c0p1 c2p0 c0p0; do
  for n in 2 4; do
    port=$((port+1))
    if [ $v = f0 ]; then E="MICS_TAIL_FUSED=0"; else E="MICS_TAIL_FUSED=1 MICS_FB_CTAS=${v:1:1} MICS_TAIL_PRIO=${v:3:1}"; fi
    env $E timeout 240 $T --nproc-per-node $n --master-port $port $B --gpus $n > gpurun_out/R2z_n${n}_$v.log 2>&1 || echo "n$n $v rc=$?"
  done
done
python tools/show.py gpurun_out/R2z_n*.log | cut -c1-300
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --compute > gpurun_out/R2z_compute_n1.log 2>&1; echo "compute rc=$?"; python tools/show.py gpurun_out/R2z_compute_n1.log | cut -c1-300
