#!/bin/bash
# bounded PDL gathers: CTAs/SM sweep for the step's per-layer gathers, N=1 and N=2, C3
cd $GRAFT_REPO_ROOT
T2="timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 1 2 3 4; do
  MICS_COPY_CTAS_PER_SM=$c timeout 200 python bench.py --no-compute > gpurun_out/r3b_c${c}_n1.log 2>&1
  MICS_COPY_CTAS_PER_SM=$c $T2 --master-port $((29630 + c)) bench.py --gpus 2 --no-compute > gpurun_out/r3b_c${c}_n2.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3b_c*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE")
PY
