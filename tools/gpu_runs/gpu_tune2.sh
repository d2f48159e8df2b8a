#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in 1 2 3; do
MICS_COPY_CTAS_PER_SM=$c python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/t1_ctas$c.log 2>&1
done
