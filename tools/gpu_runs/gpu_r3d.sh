#!/bin/bash
# bounded PDL gathers: CTAs/SM sweep at N=4 (n=8 and n=4 ranks), C3
cd $GRAFT_REPO_ROOT
T4="timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for c in 1 2 4 6; do
  MICS_COPY_CTAS_PER_SM=$c $T4 --master-port $((29650 + c)) bench.py --gpus 4 --no-compute > gpurun_out/r3d_c${c}_n4.log 2>&1
  MICS_COPY_CTAS_PER_SM=$c $T4 --master-port $((29660 + c)) bench.py --gpus 4 --ranks 4 --no-compute > gpurun_out/r3d_c${c}_r4n4.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3d_c*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE")
PY
