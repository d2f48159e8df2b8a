#!/bin/bash
cd $GRAFT_REPO_ROOT
MICS_CE_GATHER=1 timeout 300 python -m pytest tests/test_gpu_step_compute.py -x -q > gpurun_out/o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/o_tests.log; tail -2 gpurun_out/o_tests.log
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 1; do
MICS_CE_GATHER=$c $T2 --master-port 2967$c bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/o_r2n2_ce$c.log 2>&1
MICS_CE_GATHER=$c timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e > gpurun_out/o_n1_ce$c.log 2>&1
done
MICS_CE_GATHER=1 MICS_GRAPH=0 MICS_TRACE=gpurun_out/o_trace_r2n2.csv $T2 --master-port 29679 bench.py --gpus 2 --ranks 2 --compute --no-e2e --compute-steps 2 > gpurun_out/o_tr.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/o_*_ce*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), d["clocks"]["sm_mhz"])
PY
