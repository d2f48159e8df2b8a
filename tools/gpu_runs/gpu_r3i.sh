#!/bin/bash
# ncu evidence after the bounded gather chain (single process, N=1, C3): launch list,
# k_copy DRAM traffic over one step's 200 gathers, one k_copy --set full
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compute"
timeout 300 $CMD > gpurun_out/r3i_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r3i_launches.csv $CMD > gpurun_out/r3i_ncu0.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_copy -c 200 -o gpurun_out/r3i_copy $CMD > gpurun_out/r3i_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy -s 20 -c 1 -o gpurun_out/r3i_copy_full $CMD > gpurun_out/r3i_ncu2.log 2>&1
tail -2 gpurun_out/r3i_ncu*.log; ls -la gpurun_out/r3i_*
