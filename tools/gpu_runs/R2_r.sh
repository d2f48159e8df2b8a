#!/bin/bash
# round 2, call r (2 GPUs): k_hier NVLink evidence in one process (multi-device context): timing, then ncu
cd $GRAFT_REPO_ROOT
timeout 120 python tools/ncu_hier.py api > gpurun_out/R2r_hier_api.log 2>&1; tail -1 gpurun_out/R2r_hier_api.log
timeout 300 python tools/ncu_hier.py step 13 3 > gpurun_out/R2r_hier_step.log 2>&1; tail -1 gpurun_out/R2r_hier_step.log
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:k_hier -s 40 -c 12 --csv --log-file gpurun_out/R2r_ncu_hier_step.csv python tools/ncu_hier.py step 13 1 > gpurun_out/R2r_ncu_step.log 2>&1; echo "ncu step rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:k_hier -s 4 -c 4 --csv --log-file gpurun_out/R2r_ncu_hier_api.csv python tools/ncu_hier.py api 15370400 4 > gpurun_out/R2r_ncu_api.log 2>&1; echo "ncu api rc=$?"
