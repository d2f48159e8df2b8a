#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
tail -3 gpurun_out/q_tests.log
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29691 bench.py --gpus 2 --ranks 2 --compute > gpurun_out/q_r2n2_cmp.log 2>&1
timeout 900 python bench.py > gpurun_out/q_n1.log 2>&1
python tools/show.py gpurun_out/q_n1.log
python - <<'PY'
import json
for f in ["gpurun_out/q_r2n2_cmp.log", "gpurun_out/q_n1.log"]:
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l)
            c = d.get("compute_step") or d
            dd = c.get("detail", c)
            print(f, round(c["ms_per_step"],2), round(c["value"],1), dd["overlap"], c["roofline"]["achieved"], (c.get("e2e") or {}).get("value"))
PY
