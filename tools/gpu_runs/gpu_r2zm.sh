#!/bin/bash
# full verification: GPU suite (1 GPU + multi-GPU), smoke, default bench N=1/2/4 + reference arm
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/zm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zm_tests.log; tail -3 gpurun_out/zm_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/zm_n1.log 2>&1
python bench.py --impl reference > gpurun_out/zm_ref_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29611 bench.py --gpus 2 > gpurun_out/zm_n2.log 2>&1
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29612 bench.py --gpus 4 > gpurun_out/zm_n4.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/zm_*n*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); c=d.get("compute_step") or {}
            print(f, d.get("impl","mics"), round(d["value"],1), round(d.get("ms_per_step",0),3), (d.get("roofline") or {}).get("frac"), "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "cmp", c.get("value"), c.get("ms_per_step"), d.get("clocks"))
PY
