#!/bin/bash
# round 2, call P (2 B200): the step with compute on 2 GPUs, one rank each (C3, n=2, p=2) and its cuBLAS + NCCL
# comparator — with the comparator graph-captured (side stream joined)
cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $T --nproc-per-node 2 --master-port 29998 bench.py --gpus 2 --ranks 2 --compute --steps 5 --warmup 3 --compute-steps 5 --no-e2e --no-cpu-baseline --no-collectives > gpurun_out/R2P_compute_r2n2.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/R2P_compute_r2n2.log'):
    if l.startswith('{'):
        d = json.loads(l)
        print(d['metric'], d['value'], d['ms_per_step'], d.get('clocks'))
        c = d.get('compute_step') or d
        print({k: (str(v)[:400]) for k, v in c.items() if k in ('value', 'ms_per_step', 'nccl_cublas_comparator', 'clocks', 'roofline')})
PY
