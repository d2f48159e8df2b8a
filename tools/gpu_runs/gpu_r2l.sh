#!/bin/bash
cd $GRAFT_REPO_ROOT
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 python -m pytest tests/test_gpu_step_compute.py -x -q > gpurun_out/l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l_tests.log; tail -2 gpurun_out/l_tests.log
for c in 0 8 16 32; do
MICS_COMM_SMS=$c $T2 --master-port 2966$((c % 10)) bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/l_r2n2_c$c.log 2>&1
MICS_COMM_SMS=$c timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e > gpurun_out/l_n1_c$c.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/l_*_c*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), d["clocks"]["sm_mhz"])
PY
