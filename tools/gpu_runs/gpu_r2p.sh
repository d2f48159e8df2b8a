#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 8 16 24; do
MICS_CE_GATHER=1 MICS_COMM_SMS=$c $T2 --master-port 2968$((c % 10)) bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/p_r2n2_c$c.log 2>&1
done
for c in 0 16; do
MICS_CE_GATHER=1 MICS_COMM_SMS=$c timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e > gpurun_out/p_n1_c$c.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/p_*_c*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), d["clocks"]["sm_mhz"])
PY
