#!/bin/bash
# deeper gather chains at N=4 (n=8): slots x CTAs/SM, C3
cd $GRAFT_REPO_ROOT
T4="timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for sc in "4 3" "6 1" "6 2" "8 1" "8 2"; do
  set -- $sc; i=$((i+1))
  MICS_GATHER_SLOTS=$1 MICS_COPY_CTAS_PER_SM=$2 $T4 --master-port $((29700 + i)) bench.py --gpus 4 --no-compute > gpurun_out/r3h_s$1c$2_n4.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3h_s*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE")
PY
