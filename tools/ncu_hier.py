"""K3 (`k_hier`) NVLink evidence in ONE process (ncu profiles one process): a
multi-device context (mics_init_devices) over GPUs 0 and 1 with n=4 virtual ranks,
p=4, k=2 — node peers share a GPU, the stage-1 channel pulls cross NVLink, exactly the
C4 n=8 / 4-GPU placement.  Chunk = one GPT-2 1.5B block's bf16 chunk at p=4.
Prints CUDA-event GB/s (stage-1 NVLink bytes and total bytes per launch).

    python tools/ncu_hier.py [chunk_bytes] [reps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2205_00119_b200.collectives import hierarchical_all_gather_device
    from paper_2205_00119_b200.engine import Engine
    chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 30_740_800 // 4 * 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    n, p, k = 4, 4, 2
    eng = Engine(n_ranks=n, arena_bytes=(p + 1) * chunk + (256 << 20), devices=[0, 1])
    src, out = eng.alloc(chunk), eng.alloc(p * chunk)
    for r in range(n):
        eng.generate(src, r, chunk // 2, "bf16", seed=3, step=r)
    eng.synchronize()
    ptr_s = [eng.ptr(src, r) for r in range(n)]
    ptr_o = [eng.ptr(out, r) for r in range(n)]

    def run():
        hierarchical_all_gather_device(eng, p, k, ptr_s, chunk, ptr_o)

    run()
    eng.synchronize()
    ext = torch.cuda.ExternalStream(eng.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(ext)
    for _ in range(reps):
        run()
    e1.record(ext)
    eng.synchronize()
    wall = (time.perf_counter() - t0) / reps
    ms = e0.elapsed_time(e1) / reps  # GPU 0's stream; the members meet at the launch's barriers
    # per GPU per launch: 2 local ranks x (q-1) = 1 remote stage-1 chunk each over NVLink
    nvl = 2 * (p // k - 1) * chunk
    print(json.dumps({"op": "k_hier p=4 k=2, 2 ranks/GPU on 2 GPUs (one process)", "chunk_bytes": chunk,
                      "ms": ms, "wall_ms": wall * 1e3, "nvlink_bytes_per_gpu": nvl,
                      "nvlink_GBps": nvl / ms / 1e6, "gathered_bytes_per_rank": p * chunk}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
