#!/bin/bash
# round 2, call E (4 GPUs): C4 (n=8, p=4, k=2, 4 GPUs) with K9 vs the two-kernel boundary; ncu of k_fbnd on one GPU
# (8 ranks, overlapped tail forced, every replica local: the kernel's DRAM traffic vs its algorithmic bytes)
cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C4="bench.py --workload C4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
MICS_TAIL_FUSED=1 timeout 400 $T --nproc-per-node 4 --master-port 29871 $C4 --gpus 4 > gpurun_out/R2E_c4_n4_f1.log 2>&1 || echo "c4 f1 rc=$?"
MICS_TAIL_FUSED=0 timeout 400 $T --nproc-per-node 4 --master-port 29872 $C4 --gpus 4 > gpurun_out/R2E_c4_n4_f0.log 2>&1 || echo "c4 f0 rc=$?"
python tools/show.py gpurun_out/R2E_c4*.log | cut -c1-300
B1="bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-compute --no-collectives"
MICS_TAIL_OVERLAP=1 MICS_FUSED_TAIL=0 timeout 300 python $B1 > gpurun_out/R2E_n1_tail.log 2>&1; echo "n1 tail rc=$?"
python tools/show.py gpurun_out/R2E_n1_tail.log | cut -c1-300
MICS_TAIL_OVERLAP=1 MICS_FUSED_TAIL=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fbnd -c 1 -o gpurun_out/R2E_full_fbnd python $B1 > gpurun_out/R2E_ncu_fbnd.log 2>&1; echo "ncu rc=$?"
