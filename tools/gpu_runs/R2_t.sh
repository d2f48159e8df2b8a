#!/bin/bash
# round 2, call t (1 GPU): ncu evidence of the final build — launch list of the default C3 step
# (N=1), one full capture each of the dominant kernels, and the k_hier peer-pull NVLink counters need 2 GPUs (not here)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compute"
timeout 600 $B > gpurun_out/R2t_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/R2t_launches_c3_n1.csv $B > gpurun_out/R2t_ncu_list.log 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 300 -c 1 -o gpurun_out/R2t_full_copy $B > gpurun_out/R2t_ncu_copy.log 2>&1; echo "copy rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tail -c 1 -o gpurun_out/R2t_full_tail $B > gpurun_out/R2t_ncu_tail.log 2>&1; echo "tail rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 2 -c 1 -o gpurun_out/R2t_full_reduce $B > gpurun_out/R2t_ncu_reduce.log 2>&1; echo "reduce rc=$?"
