#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_step_compute.py -x -q 2>&1 | tail -2
for bn in 256 128; do echo "== BN=$bn"; MICS_GEMM_BN=$bn timeout 300 python tools/gemm_bench.py 2>&1 | cut -c1-150; done
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29891 bench.py --gpus 4 --workload C4 --ranks 4 --steps 3 --warmup 3 --no-e2e --compute > gpurun_out/zk_c4_cmp_r4n4.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/zk_c4_cmp_r4n4.log"):
    if l.startswith("{"):
        d=json.loads(l); print("C4 compute r4n4", d["ms_per_step"], d["roofline"]["achieved"], d.get("nccl_cublas_comparator"))
PY
