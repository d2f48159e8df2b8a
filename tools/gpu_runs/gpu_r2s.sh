#!/bin/bash
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/s_topo.log 2>&1
lscpu | head -30 > gpurun_out/s_lscpu.log
for d in /sys/bus/pci/devices/*; do if [ -f $d/local_cpulist ] && grep -q 0x10de $d/vendor 2>/dev/null && grep -q 0x0302 $d/class 2>/dev/null; then echo "$d $(cat $d/local_cpulist) numa=$(cat $d/numa_node)"; fi; done > gpurun_out/s_gpus.log
T4="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for m in 0 1; do
MICS_NUMA=$m $T4 --master-port 2970$m bench.py --gpus 4 --no-compute --e2e-steps 2 > gpurun_out/s_n4_numa$m.log 2>&1
done
MICS_NUMA=1 timeout 600 python bench.py --no-compute --no-cpu-baseline > gpurun_out/s_n1_numa1.log 2>&1
cat gpurun_out/s_gpus.log; cat gpurun_out/s_topo.log | head -12; grep -i "numa\|socket\|model name" gpurun_out/s_lscpu.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/s_n*.log")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, round(d["value"]), d["e2e"])
PY
