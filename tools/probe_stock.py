"""Where does the stock (cuBLAS + NCCL) compute-step comparator spend its time?
torchrun --nproc-per-node 2 tools/probe_stock.py"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2205_00119_b200.step import workloads
    wl = workloads()["C3"]
    T, h = wl.tokens, wl.hidden
    pad = os.environ.get("PAD") == "1"
    rows = [(e // h + 7) // 8 * 8 if pad else e // h for e in wl.layer_params]
    X = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    Ws = [torch.randn(r, h, device="cuda").to(torch.bfloat16) for r in rows]
    Y = [torch.empty(T, r, dtype=torch.bfloat16, device="cuda") for r in rows]

    def t(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps, (time.perf_counter() - w0) * 1e3 / reps

    def fwd():
        for l in range(len(rows)):
            torch.matmul(X, Ws[l].t(), out=Y[l])

    def bwd():
        for l in range(len(rows)):
            torch.matmul(Y[l], Ws[l])
            torch.matmul(Y[l].t(), X)
    flops = sum(2 * T * r * h for r in rows)
    ms, wall = t(fwd)
    print(rank, f"fwd 25 layers: {ms:.2f} ms device ({flops / ms / 1e9:.0f} TF/s), {wall:.2f} ms wall", flush=True)
    ms, wall = t(bwd)
    print(rank, f"bwd 25 layers: {ms:.2f} ms device ({2 * flops / ms / 1e9:.0f} TF/s), {wall:.2f} ms wall", flush=True)
    shard = torch.randn(max(rows) * h // 2, device="cuda").to(torch.bfloat16)
    out = torch.empty(2 * shard.numel(), dtype=torch.bfloat16, device="cuda")

    def ag():
        for l in range(len(rows)):
            dist.all_gather_into_tensor(out[:rows[l] * h], shard[:rows[l] * h // 2])
    ms, wall = t(ag)
    print(rank, f"25 NCCL all_gathers: {ms:.2f} ms device, {wall:.2f} ms wall", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
