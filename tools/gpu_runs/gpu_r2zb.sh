#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/ncu_nvlink.py > gpurun_out/zb_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum.per_second --clock-control none -k regex:k_reduce -c 2 --csv --log-file gpurun_out/zb_ncu_nvlink_reduce.csv python tools/ncu_nvlink.py > gpurun_out/zb_ncu.log 2>&1
cat gpurun_out/zb_plain.log; tail -3 gpurun_out/zb_ncu.log
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/zb_ncu_nvlink_reduce.csv")))
hi=[i for i,r in enumerate(rows) if "Metric Name" in r][0]; h=rows[hi]
k=h.index("Kernel Name"); n=h.index("Metric Name"); v=h.index("Metric Value"); u=h.index("Metric Unit"); d=h.index("Device")
for r in rows[hi+1:]:
    print(r[d], r[k][:40], r[n], r[v], r[u])
PY
