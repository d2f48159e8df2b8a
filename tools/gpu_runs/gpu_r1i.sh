#!/bin/bash
# (f)1 ablations: s=1 vs s=4, 2-hop vs alternative, C5 p=8 vs p=4; plus k_adam ncu at N=1
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for sch in two_hop alternative; do
  for s in 1 4; do
    timeout 600 $B --schedule $sch --micro-steps $s > gpurun_out/j_c3_n1_${sch}_s$s.log 2>&1
    $T4 --master-port 2961$s bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --schedule $sch --micro-steps $s > gpurun_out/j_c3_n4_${sch}_s$s.log 2>&1
  done
done
for p in 8 4; do
  for sch in two_hop alternative; do
    $T4 --master-port 2962$p bench.py --gpus 4 --workload C5p8 --p $p --steps 3 --warmup 3 --no-e2e --schedule $sch > gpurun_out/j_c5_n4_p${p}_${sch}.log 2>&1
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/j_launches_c3_n1.csv $B --steps 2 --warmup 1 > gpurun_out/j_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_adam -s 2 -c 1 -o gpurun_out/prof_adam $B --steps 2 --warmup 1 > gpurun_out/j_ncu_adam.log 2>&1
ncu -i gpurun_out/prof_adam.ncu-rep --page raw --csv > gpurun_out/j_ncu_adam_raw.csv 2>&1
ncu -i gpurun_out/prof_adam.ncu-rep > gpurun_out/j_ncu_adam.txt 2>&1
for f in gpurun_out/j_c*.log; do echo "== $f"; grep -o '"value": [0-9.]*\|"ms_per_step": [0-9.]*\|"phases_ms": {[^}]*}\|"workload": "[^"]*"' $f | tr '\n' ' '; grep -i "error\|Traceback" $f | tail -2; echo; done
tail -3 gpurun_out/j_ncu_adam.log
