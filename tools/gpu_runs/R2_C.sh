#!/bin/bash
# round 2, call C (4 GPUs): K9 knobs around G=2 — block, lag, one CTA per item, groups 1/3
cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
port=29830
run() {  # name n env...
  local name=$1 n=$2; shift 2
  port=$((port+1))
  env MICS_TAIL_FUSED=1 "$@" timeout 240 $T --nproc-per-node $n --master-port $port $B --gpus $n > gpurun_out/R2C_n${n}_$name.log 2>&1 || echo "$name n$n rc=$?"
}
run f0 4 MICS_TAIL_FUSED=0
run g2b16c0 4 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=16384 MICS_FB_CTAS=0
run g2b32 4 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=32768
run g3b16 4 MICS_TAIL_GROUPS=3 MICS_FB_BLOCK=16384
run g2b16l8 4 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=16384 MICS_FB_LAG=8
run g2b16l60 4 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=16384 MICS_FB_LAG=60
run g1b16 4 MICS_TAIL_GROUPS=1 MICS_FB_BLOCK=16384
run g1b16 2 MICS_TAIL_GROUPS=1 MICS_FB_BLOCK=16384
run g2b8 2 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=8192
run g2b32 2 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=32768
run g3b16 2 MICS_TAIL_GROUPS=3 MICS_FB_BLOCK=16384
run g2b16c0 2 MICS_TAIL_GROUPS=2 MICS_FB_BLOCK=16384 MICS_FB_CTAS=0
python tools/show.py gpurun_out/R2C_n*.log | cut -c1-200
