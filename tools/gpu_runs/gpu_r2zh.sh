#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/zh_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/zh_mgpu.log; tail -4 gpurun_out/zh_mgpu.log
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 0 1; do
MICS_CE_RS=$c $T2 --master-port 2985$c bench.py --gpus 2 --ranks 2 --compute --no-e2e > gpurun_out/zh_r2n2_ce$c.log 2>&1
done
rm -f gpurun_out/zh_trace*
MICS_GRAPH=0 MICS_TRACE=gpurun_out/zh_trace.csv $T2 --master-port 29859 bench.py --gpus 2 --ranks 2 --compute --no-e2e --compute-steps 2 > gpurun_out/zh_tr.log 2>&1
python tools/trace_report.py gpurun_out/zh_trace.csv.0 0 | head -5
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/zh_r2n2*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), round(d["value"],1), "serial", round(dd["serialised_ms"],2), {k: round(v,3) if v else v for k,v in dd["overlap"].items()}, "gemmTF", round(d["roofline"]["achieved"]), d["clocks"]["sm_mhz"], (d.get("nccl_cublas_comparator") or {}).get("ms_per_step"))
PY
