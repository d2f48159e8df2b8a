#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k_tests.log
timeout 600 python bench.py --compute --no-cpu-baseline > gpurun_out/k_c3_cmp_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29652 bench.py --gpus 2 --ranks 2 --compute > gpurun_out/k_c3_cmp_r2n2.log 2>&1
tail -3 gpurun_out/k_tests.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/k_c3*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), dd["overlap"], "gemmTF", round(d["roofline"]["achieved"]), d["roofline"]["frac"], d["clocks"], "e2e", d["e2e"]["value"])
PY
