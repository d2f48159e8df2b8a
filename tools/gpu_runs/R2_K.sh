#!/bin/bash
# round 2, call K (4 B200): one rank per GPU (the N=8 regime: partition groups across GPUs) — gather chain
# knobs: in-flight gathers (MICS_GATHER_SLOTS) x CTAs per SM of the chained gathers (MICS_COPY_CTAS_PER_SM)
cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives --gpus 4 --ranks 4"
port=29980
for v in s3c3 s6c3 s3c2 s3c4 s6c4 s12c3; do
  s=${v#s}; s=${s%c*}; c=${v#*c}
  port=$((port+1))
  MICS_GATHER_SLOTS=$s MICS_COPY_CTAS_PER_SM=$c timeout 240 $T --nproc-per-node 4 --master-port $port $B > gpurun_out/R2K_r4n4_$v.log 2>&1 || echo "$v rc=$?"
done
python tools/show.py gpurun_out/R2K_*.log | cut -c1-200
