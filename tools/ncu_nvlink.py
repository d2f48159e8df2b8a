"""Single-process NVLink evidence for ncu (which profiles one process only): libmics'
own collective kernels on GPU 0 pulling a peer rank's buffer that lives on GPU 1
(peer access enabled), so `nvlrx__bytes` / `nvltx__bytes` of k_copy and k_reduce can
be captured.  n = 2 ranks in one context on GPU 0; rank 1's source is GPU 1 memory.

    python tools/ncu_nvlink.py            (2 GPUs; prints CUDA-event GB/s per op)
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2205_00119_b200.collectives import all_gather_device, reduce_scatter_device
    from paper_2205_00119_b200.engine import Engine
    torch.cuda.set_device(0)
    cudart = C.CDLL("libcudart.so.12")
    for dev, peer in ((0, 1), (1, 0)):
        cudart.cudaSetDevice(dev)
        r = cudart.cudaDeviceEnablePeerAccess(peer, 0)
        assert r in (0, 704), r  # 704 = already enabled
    cudart.cudaSetDevice(0)
    chunk = 512 << 20  # bytes per position: 1 GiB gathered, 1 GiB reduce-scatter input per rank
    eng = Engine(n_ranks=2, device=0, arena_bytes=11 * chunk + (64 << 20))
    ext = torch.cuda.ExternalStream(eng.stream())
    src0 = eng.alloc(chunk)
    out = eng.alloc(2 * chunk)
    rs_in0 = eng.alloc(2 * chunk)
    src1 = torch.randint(0, 255, (chunk,), dtype=torch.uint8, device="cuda:1")
    rs_in1 = torch.randn(2 * chunk // 4, device="cuda:1")
    torch.cuda.synchronize(1)
    res = []

    def timed(name, fn, nvl_bytes, reps=10):
        fn()
        eng.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(reps):
            fn()
        e1.record(ext)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res.append({"op": name, "ms": ms, "nvlink_bytes": nvl_bytes, "nvlink_GBps": nvl_bytes / ms / 1e6})
    # all-gather p=2: rank 1's chunk crosses NVLink once (one read feeds both local outputs)
    timed("k_copy all_gather p=2, peer source on GPU1",
          lambda: all_gather_device(eng, [0, 1], [eng.ptr(src0, 0), src1.data_ptr()], chunk,
                                    [eng.ptr(out, 0), eng.ptr(out, 1)]), chunk)
    # reduce-scatter p=2 fp32: rank 1's whole input (both halves) crosses NVLink
    elems = 2 * chunk // 4
    timed("k_reduce reduce_scatter p=2 f32, peer input on GPU1",
          lambda: reduce_scatter_device(eng, [0, 1], [eng.ptr(rs_in0, 0), rs_in1.data_ptr()], elems,
                                        [eng.ptr(out, 0), eng.ptr(out, 1)]), 2 * chunk)
    for r in res:
        print(json.dumps(r), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
