#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/zt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zt_tests.log; tail -3 gpurun_out/zt_tests.log
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T4 --master-port 29941 bench.py --gpus 4 --ranks 4 > gpurun_out/zt_r4n4.log 2>&1
python tools/show.py gpurun_out/zt_r4n4.log | cut -c1-230
