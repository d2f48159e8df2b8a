"""C2 (BASELINE.json configs[1]): partition-group all-gather + reduce-scatter sweep,
1 MiB..1 GiB gathered bytes per rank, p in {2,4,8} (<= GPUs), one rank per GPU, all
n/p groups concurrent — libmics (persistent plans) vs NCCL on split communicators.

    torchrun --nproc-per-node N bench.py --gpus N --sweep [--steps K]

busBW = (p-1) * M / p / t per rank; one JSON line per point, times are
CUDA-event averages over back-to-back calls (median of 3 trials), max over ranks.
NCCL's calls are captured in a CUDA graph and replayed (no per-call host launch in
the timed region), like libmics' persistent plans.
"""
from __future__ import annotations

import json
import os
import statistics

NVLINK = 770.0


def _time(fn, stream_ext, reps, world, gloo, trials=3):
    """nccl-tests style: `reps` back-to-back calls between two events (per-call host
    skew between ranks amortises), median over trials, max over ranks."""
    import torch
    import torch.distributed as dist

    import bench
    ts = []
    for _ in range(trials):
        bench.barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream_ext)
        fn(reps)
        e1.record(stream_ext)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    t = statistics.median(ts)
    if world > 1:
        x = torch.tensor([t], dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX, group=gloo)
        t = float(x.item())
    return t * 1e3  # us


def nccl_runner(call, reps, world):
    """NCCL timed without host launch cost: `reps` back-to-back calls captured once in
    a CUDA graph (torch.cuda.graph) and replayed, as libmics replays its persistent
    plans.  Returns (fn(k) running the reps calls, "cuda_graph"), or the eager loop
    ("eager") when the capture is refused."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up (communicator setup) outside the capture
        for _ in range(3):
            call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                call()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        return (lambda k: g.replay()), "cuda_graph"
    except Exception:  # noqa: BLE001  (capture unsupported on this stack: time the eager loop)
        torch.cuda.synchronize()
        return (lambda k: [call() for _ in range(k)]), "eager"


def run_sweep(args, rank, world, local, sizes=None, quiet=False):
    """All-gather / reduce-scatter busBW (libmics plans and NCCL) for every p in {2,4,8}
    dividing `world`, one rank per GPU; prints one JSON line per point unless `quiet`;
    returns the points."""
    import torch
    import torch.distributed as dist

    import bench
    from paper_2205_00119_b200 import dist as mdist
    from paper_2205_00119_b200.collectives import RS_STORE, plan_all_gather, plan_reduce_scatter
    from paper_2205_00119_b200.engine import Engine

    gloo = bench.GLOO
    if sizes is None:
        maxlog = int(os.environ.get("MICS_SWEEP_MAXLOG", 30))
        sizes = [1 << e for e in range(20, maxlog + 1)]
    M = max(sizes)
    eng = Engine(n_ranks=world, world=world, world_rank=rank, device=local, arena_bytes=3 * M + (64 << 20))
    mdist.connect(eng, gloo)
    src, dst = eng.alloc(M), eng.alloc(M)
    eng.generate(src, rank, M // 4, "f32", seed=rank)
    eng.synchronize()
    ext = torch.cuda.ExternalStream(eng.stream())
    dev = torch.device("cuda", local)
    t_in = torch.randn(M // 4, device=dev)
    t_out = torch.empty(M // 4, device=dev)
    results = []
    for p in (2, 4, 8):
        if p > world or world % p:
            continue
        g = rank // p
        ranks = list(range(g * p, (g + 1) * p))
        groups = [dist.new_group(list(range(h * p, (h + 1) * p))) for h in range(world // p)] if world > 1 else []
        pg = groups[g] if groups else None
        for m in sizes:
            reps = 20 if m <= (64 << 20) else 5
            chunk = m // p
            ag = plan_all_gather(eng, ranks, [eng.ptr(src, r) for r in ranks], chunk, [eng.ptr(dst, r) for r in ranks])
            rs = plan_reduce_scatter(eng, ranks, [eng.ptr(src, r) for r in ranks], m // 4,
                                     [eng.ptr(dst, r) for r in ranks], "f32", mode=RS_STORE)
            for plan, op in ((ag, "allgather"), (rs, "reducescatter")):
                plan.run(3)
                eng.synchronize()
                bench.barrier(world)
                us = _time(plan.run, ext, reps, world, gloo)
                nmode = None
                if pg is not None:
                    a_in, a_out = t_in.view(torch.uint8)[:chunk], t_out.view(torch.uint8)[:m]
                    r_in, r_out = t_in[:m // 4], t_out[:m // 4 // p]
                    nccl = (lambda: dist.all_gather_into_tensor(a_out, a_in, group=pg)) if op == "allgather" else \
                        (lambda: dist.reduce_scatter_tensor(r_out, r_in, group=pg))
                    run, nmode = nccl_runner(nccl, reps, world)
                    bench.barrier(world)
                    nus = _time(run, torch.cuda.current_stream(), reps, world, gloo)
                else:
                    nus = None
                bus = (p - 1) * m / p / (us * 1e-6) / 1e9
                line = {"sweep": "C2", "op": op, "p": p, "gpus": world, "bytes": m, "mics_us": us,
                        "mics_busbw_GBps": bus, "frac_nvlink_770": bus / NVLINK,
                        "nccl_us": nus, "nccl_busbw_GBps": (p - 1) * m / p / (nus * 1e-6) / 1e9 if nus else None,
                        "nccl_launch": nmode}
                results.append(line)
                if rank == 0 and not quiet:
                    print(json.dumps(line), flush=True)
            ag.close()
            rs.close()
    if rank == 0 and results and not quiet:
        big = [r for r in results if r["bytes"] >= (256 << 20)]
        wins = sum(1 for r in results if r["nccl_us"] and r["mics_us"] < r["nccl_us"])
        print(json.dumps({"sweep_summary": "C2", "points": len(results), "beats_nccl": wins,
                          "min_frac_nvlink_>=256MiB": min(r["frac_nvlink_770"] for r in big) if big else None}),
              flush=True)
    eng.close()
    return results
