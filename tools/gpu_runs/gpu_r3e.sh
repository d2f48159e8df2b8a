#!/bin/bash
# gather slots (in-flight bound) x CTAs/SM at N=4 (n=8 and n=4 ranks), C3; step tests first
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step.py -q -m gpu > gpurun_out/r3e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_tests.log; tail -2 gpurun_out/r3e_tests.log
T4="timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for sc in "3 1" "3 2" "3 3" "4 1" "4 2"; do
  set -- $sc; i=$((i+1))
  MICS_GATHER_SLOTS=$1 MICS_COPY_CTAS_PER_SM=$2 $T4 --master-port $((29670 + i)) bench.py --gpus 4 --no-compute > gpurun_out/r3e_s$1c$2_n4.log 2>&1
  MICS_GATHER_SLOTS=$1 MICS_COPY_CTAS_PER_SM=$2 $T4 --master-port $((29680 + i)) bench.py --gpus 4 --ranks 4 --no-compute > gpurun_out/r3e_s$1c$2_r4n4.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3e_s*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE")
PY
