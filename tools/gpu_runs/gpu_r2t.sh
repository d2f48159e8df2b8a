#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for f in 0 40; do for c in 16 24; do
MICS_RS_SMEM_FLOOR=$f MICS_COMM_SMS=$c $T2 --master-port $((29700 + c + f)) bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/t_r2n2_f${f}_c$c.log 2>&1
done; done

python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), d["clocks"]["sm_mhz"])
PY
