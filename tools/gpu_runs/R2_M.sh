#!/bin/bash
# round 2, call M (4 B200): C5 (10B, bf16 grads generated in-step, n=8) at p=4 (K9 boundary) and p=8 (ZeRO-3)
cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-compute --no-collectives --workload C5p8"
timeout 900 $T --nproc-per-node 4 --master-port 29991 $B --p 4 > gpurun_out/R2M_c5p4_n4.log 2>&1; echo "p4 rc=$?"
timeout 900 $T --nproc-per-node 4 --master-port 29992 $B > gpurun_out/R2M_c5p8_n4.log 2>&1; echo "p8 rc=$?"
python tools/show.py gpurun_out/R2M_*.log | cut -c1-300
