#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compute"
timeout 300 $CMD > gpurun_out/zza_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_copy -c 200 -o gpurun_out/zza_copy $CMD > gpurun_out/zza_ncu1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tail -c 1 -o gpurun_out/zza_tail $CMD > gpurun_out/zza_ncu2.log 2>&1
tail -2 gpurun_out/zza_ncu1.log gpurun_out/zza_ncu2.log 2>/dev/null | tail -4; ls -la gpurun_out/zza_*
