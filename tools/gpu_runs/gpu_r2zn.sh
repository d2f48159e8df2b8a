#!/bin/bash
cd $GRAFT_REPO_ROOT
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
( time $T4 --master-port 29612 bench.py --gpus 4 ) > gpurun_out/zn_n4.log 2>&1
grep real gpurun_out/zn_n4.log
python - <<'PY'
import json
for l in open("gpurun_out/zn_n4.log"):
    if l.startswith("{"):
        d=json.loads(l); print(d["value"], json.dumps(d.get("collectives")))
PY
