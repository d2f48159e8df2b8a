#!/bin/bash
# pipelined boundary (MICS_PIPELINE=1) vs default overlapped tail at N=4, C3
cd $GRAFT_REPO_ROOT
T4="timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
MICS_PIPELINE=1 $T4 --master-port 29721 bench.py --gpus 4 --no-compute > gpurun_out/r3k_pipe_n4.log 2>&1
MICS_PIPELINE=1 $T4 --master-port 29722 bench.py --gpus 4 --ranks 4 --no-compute > gpurun_out/r3k_pipe_r4n4.log 2>&1
$T4 --master-port 29723 bench.py --gpus 4 --no-compute > gpurun_out/r3k_def_n4.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r3k_*.log")):
    ok=False
    for l in open(f):
        if l.startswith("{"):
            ok=True; d=json.loads(l)
            print(f, round(d["value"],1), round(d["ms_per_step"],3), d["phases_ms"], d.get("clocks",{}).get("sm_mhz"))
    if not ok: print(f, "NO LINE"); print(open(f).read()[-600:])
PY
