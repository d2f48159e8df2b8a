#!/bin/bash
# the driver's round-end invocations (default flags) at N=1,2,4 + reference arm
cd $GRAFT_REPO_ROOT
( time python bench.py ) > gpurun_out/r_n1.log 2>&1
( time python bench.py --impl reference ) > gpurun_out/r_ref_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
( time $T2 --master-port 29611 bench.py --gpus 2 ) > gpurun_out/r_n2.log 2>&1
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
( time $T4 --master-port 29612 bench.py --gpus 4 ) > gpurun_out/r_n4.log 2>&1
( time $T4 --master-port 29613 bench.py --gpus 4 --ranks 4 ) > gpurun_out/r_r4n4.log 2>&1
( time $T4 --master-port 29614 bench.py --gpus 4 --impl reference ) > gpurun_out/r_ref_n4.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1
python tools/show.py gpurun_out/r_n*.log gpurun_out/r_r4n4.log
grep real gpurun_out/r_*.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l)
            c=d.get("compute_step") or {}
            print(f, d.get("impl"), round(d["value"],1), "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "cmp", c.get("value"), c.get("ms_per_step"), (c.get("overlap") or {}).get("hidden_comm_frac"), d.get("clocks"))
PY
tail -2 gpurun_out/r_smoke.log
