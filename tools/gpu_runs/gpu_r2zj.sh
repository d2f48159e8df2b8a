#!/bin/bash
# every BASELINE config on 4 GPUs with the current code: communication step and step with compute
cd $GRAFT_REPO_ROOT
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29881 bench.py --gpus 4 --workload C1 --steps 20 --no-e2e > gpurun_out/zj_c1_n4.log 2>&1
$T --master-port 29882 bench.py --gpus 4 --workload C4 --steps 3 --warmup 3 --no-e2e > gpurun_out/zj_c4_n4.log 2>&1
$T --master-port 29883 bench.py --gpus 4 --workload C4 --ranks 4 --steps 3 --warmup 3 --no-e2e > gpurun_out/zj_c4_r4n4.log 2>&1
$T --master-port 29884 bench.py --gpus 4 --workload C5p8 --steps 2 --warmup 3 --no-e2e --no-compute > gpurun_out/zj_c5p8_n4.log 2>&1
$T --master-port 29885 bench.py --gpus 4 --workload C5p8 --p 4 --steps 2 --warmup 3 --no-e2e --no-compute > gpurun_out/zj_c5p4_n4.log 2>&1
$T --master-port 29886 bench.py --gpus 4 --ranks 4 --workload C3 --compute --no-e2e > gpurun_out/zj_c3_cmp_r4n4.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/zj_*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True
            d=json.loads(l); c=d.get("compute_step") or {}
            det=d.get("detail") or {}
            print(f, d["config"]["workload"], "| ms", round(d["ms_per_step"],3), "| samples/s", round(d["value"],1),
                  "| roof", d["roofline"]["bound"], round(d["roofline"]["frac"],3), "| phases", {k: round(v,2) for k,v in (d.get("phases_ms") or {}).items()},
                  "| nccl", (d.get("nccl_comparator") or {}).get("ms_per_step"), (d.get("nccl_cublas_comparator") or {}).get("ms_per_step"),
                  "| cmp", c.get("ms_per_step"), (c.get("nccl_cublas_comparator") or {}).get("ms_per_step"), (det.get("overlap") or {}))
    if not ok: print(f, "NO LINE"); import subprocess; print(open(f).read()[-800:])
PY
