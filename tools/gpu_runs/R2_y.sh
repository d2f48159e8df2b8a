#!/bin/bash
# round 2, call y (4 GPUs): K9 grid (CTAs per SM 1 vs 2) and the two-kernel boundary, N=2 and N=4, twice each
cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
port=29750
for rep in 1 2; do
for v in f0 f1c1 f1c2; do
  for n in 2 4; do
    port=$((port+1))
    f=${v:1:1}; c=${v:3:1}; [ -z "$c" ] && c=2
    MICS_TAIL_FUSED=$f MICS_FB_CTAS=$c timeout 240 $T --nproc-per-node $n --master-port $port $B --gpus $n > gpurun_out/R2y_n${n}_${v}_$rep.log 2>&1 || echo "n$n $v rc=$?"
  done
done
done
python tools/show.py gpurun_out/R2y_n*.log | cut -c1-330
