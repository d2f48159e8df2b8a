#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/zi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zi_tests.log; tail -2 gpurun_out/zi_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/zi_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29871 bench.py --gpus 2 > gpurun_out/zi_n2.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/zi_n*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); c=d.get("compute_step") or {}
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["roofline"]["frac"], "e2e", round(d["e2e"]["value"],1), "cmp", round(c.get("value",0),1), c.get("ms_per_step"), d["clocks"])
PY
