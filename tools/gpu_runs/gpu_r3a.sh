#!/bin/bash
# PDL rule for independent gathers: one thread per CTA waits for the predecessor before
# triggering (bounds in-flight gathers to two); step tests + bench N=1/2 (bounded timeouts)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_multigpu.py -q -m gpu > gpurun_out/r3a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_tests.log; tail -3 gpurun_out/r3a_tests.log
timeout 300 python bench.py --no-compute > gpurun_out/r3a_n1.log 2>&1
T2="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29621 bench.py --gpus 2 --no-compute > gpurun_out/r3a_n2.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3a_n*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE")
PY
