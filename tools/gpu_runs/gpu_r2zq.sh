#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/zq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zq_tests.log; tail -3 gpurun_out/zq_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/zq_n1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/zq_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compute > gpurun_out/zq_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 1 -c 1 -o gpurun_out/zq_tail python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compute > gpurun_out/zq_ncu2.log 2>&1
python tools/show.py gpurun_out/zq_n1.log | cut -c1-300
tail -2 gpurun_out/zq_ncu.log gpurun_out/zq_ncu2.log
