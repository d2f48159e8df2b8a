"""Small-message latency probe: back-to-back replays of a tiny all-gather plan and
of the device flag barrier, one rank per GPU (or 2 ranks on one GPU when world=1).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/latency.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2205_00119_b200 import dist as mdist
    from paper_2205_00119_b200.collectives import RS_STORE, plan_all_gather, plan_reduce_scatter
    from paper_2205_00119_b200.engine import Engine

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    n = max(2, world)
    eng = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=64 << 20)
    if world > 1:
        mdist.connect(eng)
    src, dst = eng.alloc(8 << 20), eng.alloc(16 << 20)
    ext = torch.cuda.ExternalStream(eng.stream())
    ranks = list(range(n))
    reps = int(os.environ.get("REPS", 200))

    host = {}

    def timeit(fn, key=None):
        best = 1e9
        for _ in range(3):
            eng.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            h0 = time.perf_counter()
            fn()
            h1 = time.perf_counter()
            e1.record(ext)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
            if key:
                host[key] = min(host.get(key, 1e9), (h1 - h0) * 1e6 / reps)
        if world > 1:
            x = torch.tensor([best], dtype=torch.float64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            best = float(x.item())
        return best

    out = {"world": world, "n": n, "pdl": os.environ.get("MICS_PDL", "1")}
    out["barrier_us"] = timeit(lambda: [eng.barrier() for _ in range(reps)], "barrier")
    for b in (16, 4096, 1 << 16, 1 << 20):
        ag = plan_all_gather(eng, ranks, [eng.ptr(src, r) for r in ranks], b // n,
                             [eng.ptr(dst, r) for r in ranks])
        out[f"ag_{b}_us"] = timeit(lambda: ag.run(reps), f"ag_{b}")
        ag.close()
        rs = plan_reduce_scatter(eng, ranks, [eng.ptr(src, r) for r in ranks], max(n, b // 4),
                                 [eng.ptr(dst, r) for r in ranks], "f32", mode=RS_STORE)
        out[f"rs_{b}_us"] = timeit(lambda: rs.run(reps), f"rs_{b}")
        rs.close()
    out["host_enqueue_us"] = host
    if rank == 0:
        print(json.dumps(out), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
