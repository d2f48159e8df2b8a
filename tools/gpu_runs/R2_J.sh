#!/bin/bash
# round 2, call J (4 B200): the whole GPU suite and smoke on the final tree (after the K10 removal, the K9
# simplification and the full-size every-element tests), plus the driver's N=1 bench command
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/R2J_tests.log 2>&1; echo "rc=$?" >> gpurun_out/R2J_tests.log; tail -4 gpurun_out/R2J_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/R2J_smoke.log 2>&1; tail -1 gpurun_out/R2J_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/R2J_n1.log 2>&1; echo "n1 rc=$?"
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $T --nproc-per-node 2 --master-port 29971 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/R2J_n2.log 2>&1; echo "n2 rc=$?"
timeout 900 $T --nproc-per-node 4 --master-port 29972 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/R2J_n4.log 2>&1; echo "n4 rc=$?"
python tools/show.py gpurun_out/R2J_n*.log | cut -c1-260
