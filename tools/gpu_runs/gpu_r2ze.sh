#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for o in 1 0; do
MICS_RS_OVERLAP=$o $T2 --master-port 2984$o bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/ze_r2n2_o$o.log 2>&1
MICS_RS_OVERLAP=$o timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e > gpurun_out/ze_n1_o$o.log 2>&1
done
MICS_RS_OVERLAP=0 timeout 300 python -m pytest tests/test_gpu_step_compute.py -x -q 2>&1 | tail -1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/ze_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), d["clocks"]["sm_mhz"], (d.get("nccl_cublas_comparator") or {}).get("ms_per_step"))
PY
