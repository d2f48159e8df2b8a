#!/bin/bash
# MICS_GATHER_CTR=1 (device slot counters instead of fences): step tests, then C3 bench A/B
cd $GRAFT_REPO_ROOT
MICS_GATHER_CTR=1 timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_multigpu.py -x -q -m gpu > gpurun_out/r3l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3l_tests.log; tail -3 gpurun_out/r3l_tests.log
grep -q "rc=0" gpurun_out/r3l_tests.log || exit 1
MICS_GATHER_CTR=1 timeout 200 python bench.py --no-compute > gpurun_out/r3l_ctr_n1.log 2>&1
T4="timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for c in 1 3; do
  MICS_GATHER_CTR=1 MICS_COPY_CTAS_PER_SM=$c $T4 --master-port $((29730 + c)) bench.py --gpus 4 --no-compute > gpurun_out/r3l_ctr_c${c}_n4.log 2>&1
  MICS_GATHER_CTR=1 MICS_COPY_CTAS_PER_SM=$c $T4 --master-port $((29740 + c)) bench.py --gpus 4 --ranks 4 --no-compute > gpurun_out/r3l_ctr_c${c}_r4n4.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3l_ctr*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE"); print(open(f).read()[-400:])
PY
