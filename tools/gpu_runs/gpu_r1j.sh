#!/bin/bash
# C2 sweep with back-to-back (nccl-tests style) timing, 4 GPUs
cd $GRAFT_REPO_ROOT
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29631 bench.py --gpus 4 --sweep > gpurun_out/k_sweep_n4.log 2>&1
grep -E '^\{' gpurun_out/k_sweep_n4.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if 'op' in d: print(d['op'][:6], d['p'], d['bytes'] >> 20, 'MiB', round(d['mics_us'], 1), 'us', round(d['mics_busbw_GBps']), 'GB/s  nccl', round(d['nccl_us'], 1), round(d['nccl_busbw_GBps']))
    else: print(d)
"
