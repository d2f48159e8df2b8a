"""Summarise a MICS_TRACE timeline (`<path>.<process>`: a `step` marker row, then one
row per gather / GEMM group / reduce-scatter / boundary of that step).

    python tools/trace_report.py trace.csv [rank]

Prints, for the last traced step: total span, GEMM busy time, time the GEMM
stream idled waiting (gaps between GEMM groups), gather durations alone vs while
a GEMM ran, and the reduce-scatter / boundary tail.
"""
import sys


def main():
    path = sys.argv[1]
    want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    steps, cur = [], []
    for ln in open(path):
        rk, op, t, l, a, b = ln.strip().split(",")
        if int(rk) != want:
            continue
        if op == "step":  # csrc/step.cpp writes one marker row per traced step
            if cur:
                steps.append(cur)
            cur = []
            continue
        cur.append((op, int(t), int(l), float(a), float(b)))
    steps.append(cur)
    ops = steps[-1]
    t0 = min(o[3] for o in ops)
    span = max(o[4] for o in ops) - t0
    gem = sorted([o for o in ops if o[0] in ("fwd", "bwd")], key=lambda o: o[3])
    busy = sum(o[4] - o[3] for o in gem)
    gaps = []
    for x, y in zip(gem, gem[1:]):
        if y[3] > x[4] + 1e-3:
            gaps.append((y[3] - x[4], y[0], y[1], y[2]))
    gat = [o for o in ops if o[0] == "gather"]
    rs = [o for o in ops if o[0] == "rs"]
    bnd = [o for o in ops if o[0] == "boundary"]
    print(f"steps traced {len(steps)}; last step span {span:.3f} ms; GEMM busy {busy:.3f} ms "
          f"({len(gem)} groups); GEMM-stream gaps {sum(g[0] for g in gaps):.3f} ms in {len(gaps)} gaps")
    print(f"gathers: {len(gat)}, total {sum(o[4] - o[3] for o in gat):.3f} ms, "
          f"mean {sum(o[4] - o[3] for o in gat) / max(1, len(gat)) * 1e3:.1f} us")
    print("rs:", [(o[1], round(o[3] - t0, 3), round(o[4] - o[3], 3)) for o in rs])
    print("boundary:", [(round(o[3] - t0, 3), round(o[4] - o[3], 3)) for o in bnd])
    print("largest GEMM-stream gaps (ms, before op t l):", sorted(gaps, reverse=True)[:10])
    print("first 12 ops:")
    for o in sorted(ops, key=lambda o: o[3])[:12]:
        print(f"  {o[0]:8s} t={o[1]} l={o[2]:3d} {o[3] - t0:9.3f} .. {o[4] - t0:9.3f}  ({(o[4] - o[3]) * 1e3:8.1f} us)")


if __name__ == "__main__":
    main()
