#!/bin/bash
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/i_trace_*
T2="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for g in 0 1; do
MICS_GRAPH=$g timeout 600 python bench.py --compute --no-cpu-baseline --no-e2e --compute-steps 3 > gpurun_out/i_c3_cmp_n1_g$g.log 2>&1
MICS_GRAPH=$g $T2 --master-port 2965$g bench.py --gpus 2 --ranks 2 --compute --no-e2e --compute-steps 3 > gpurun_out/i_c3_cmp_r2n2_g$g.log 2>&1
done
MICS_GRAPH=0 MICS_TRACE=gpurun_out/i_trace_r2n2.csv $T2 --master-port 29659 bench.py --gpus 2 --ranks 2 --compute --no-e2e --compute-steps 2 > gpurun_out/i_c3_cmp_r2n2_tr.log 2>&1
python tools/trace_report.py gpurun_out/i_trace_r2n2.csv.0 0
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/i_c3*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); dd=d["detail"]
            print(f, round(d["ms_per_step"],2), "serial", round(dd["serialised_ms"],2), "gemm", round(dd["serialised_phases_ms"]["gemm_ms"],1), d["clocks"]["sm_mhz"])
PY
