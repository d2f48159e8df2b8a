#!/bin/bash
cd $GRAFT_REPO_ROOT
PAD=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29791 tools/probe_stock.py 2>&1 | grep "^0 "
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29781 bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/za_r2n2_cmp.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/za_r2n2_cmp.log"):
    if l.startswith("{"):
        d=json.loads(l); print("mics", d["ms_per_step"], d["value"], "stock", d["nccl_cublas_comparator"])
PY
