#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/x_tests.log 2>&1; echo "rc=$?" >> gpurun_out/x_tests.log; tail -3 gpurun_out/x_tests.log
timeout 600 python bench.py --compute --no-cpu-baseline > gpurun_out/x_c3_cmp_n1.log 2>&1
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T2 --master-port 29741 bench.py --gpus 2 --ranks 2 --compute > gpurun_out/x_c3_cmp_r2n2.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/x_c3*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"], "e2e", round(d["e2e"]["value"],1))
PY
