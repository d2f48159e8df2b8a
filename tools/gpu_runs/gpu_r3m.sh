#!/bin/bash
# final verification of the round (bounded timeouts)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log; tail -3 gpurun_out/r3m_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py > gpurun_out/r3m_n1.log 2>&1
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29751 bench.py --gpus 2 > gpurun_out/r3m_n2.log 2>&1
T4="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29752 bench.py --gpus 4 > gpurun_out/r3m_n4.log 2>&1
$T4 --master-port 29753 bench.py --gpus 4 --ranks 4 > gpurun_out/r3m_r4n4.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3m_*n*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l); c=d.get("compute_step") or {}
            print(f, round(d["value"],1), round(d.get("ms_per_step",0),3), d["roofline"]["phase"], round(d["roofline"]["frac"],3), "e2e", round((d.get("e2e") or {}).get("value",0),1), "cmp", c.get("value"), "coll", len(d.get("collectives") or []), d.get("clocks",{}).get("sm_mhz"), d.get("phases_ms"))
    if not ok: print(f, "NO LINE")
PY
