#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e > gpurun_out/h_c3_cmp_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29652 bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/h_c3_cmp_r2n2.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/h_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), "serial", round(dd["serialised_ms"],2), dd["overlap"], "gemmTF", round(d["roofline"]["achieved"]), d["clocks"])
PY
