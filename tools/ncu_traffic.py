"""Average dram__bytes_read.sum + dram__bytes_write.sum per launch from an ncu report,
and merge it into profiles/ncu_traffic.json under key "<workload>|<n_gpus>|<phase>"."""
import csv
import io
import json
import os
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
ti = h.index("gpu__time_duration.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tsc = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1}
vals, times = [], []
for r in rows[2:]:
    vals.append(float(r[ri].replace(",", "")) * scale[units[ri]] + float(r[wi].replace(",", "")) * scale[units[wi]])
    times.append(float(r[ti].replace(",", "")) * tsc.get(units[ti], 1))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
table = json.load(open(path)) if os.path.exists(path) else {}
table[key] = {"dram_bytes_per_launch": sum(vals) / len(vals), "launches": len(vals),
              "ncu_time_s_per_launch": sum(times) / len(times), "report": os.path.basename(rep)}
json.dump(table, open(path, "w"), indent=1, sort_keys=True)
print(key, table[key])
