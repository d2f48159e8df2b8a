"""Summarise bench / sweep JSON lines from log files."""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith('{'):
            continue
        d = json.loads(l)
        if 'sweep' in d:
            n = d.get('nccl_us')
            print(f"{d['op']:14s} p={d['p']} {d['bytes'] >> 20:5d}MiB mics {d['mics_us']:9.1f}us "
                  f"{d['mics_busbw_GBps']:6.1f}GB/s ({d['frac_nvlink_770']:.2f})  nccl "
                  f"{(n or 0):9.1f}us {(d['nccl_busbw_GBps'] or 0):6.1f}")
        elif 'sweep_summary' in d:
            print(d)
        elif 'metric' in d:
            r = d.get('roofline') or {}
            print(f, f"ms/step={d['ms_per_step']:.3f} value={d['value']:.1f} phases={d.get('phases_ms')} "
                     f"roof={r.get('bound')} {r.get('frac', 0):.3f} kernel={r.get('kernel')} "
                     f"nccl={(d.get('nccl_comparator') or {}).get('ms_per_step')} e2e={(d.get('e2e') or {}).get('value')}")
