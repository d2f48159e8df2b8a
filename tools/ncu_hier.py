"""K3 (`k_hier`) NVLink evidence in ONE process (ncu profiles one process): a
multi-device context (mics_init_devices) over GPUs 0 and 1.

  python tools/ncu_hier.py api  [chunk] [reps]   one hierarchical_all_gather per call (per-visit
                                                 k_hier, entry/exit barrier), n=4, p=4, k=2
  python tools/ncu_hier.py step [layers] [steps] the comm-only MiCS step on GPT-2 1.5B layers
                                                 (C4 shapes), n=4 ranks, p=4, k=2: merged k_hier
                                                 launches (stage 1 of 3 visits + stage 3 of the
                                                 previous 3, done counters)

  python tools/ncu_hier.py peer [chunk] [reps]  ncu-friendly: one GPU context (ncu replays
                                                 kernels one at a time, so kernels that wait
                                                 on another GPU's kernels cannot be profiled);
                                                 the channel peers' shards live on GPU 1

All place node peers on one GPU and the stage-1 channel across NVLink, exactly the C4
n=8 / 4-GPU placement.  Prints CUDA-event times and the NVLink bytes per launch.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2205_00119_b200.engine import Engine
    mode = sys.argv[1] if len(sys.argv) > 1 else "api"
    torch.cuda.set_device(0)
    if mode == "step":
        import bench
        from paper_2205_00119_b200.step import MicsStep, StepOptions
        from paper_2205_00119_b200.workloads import Workload, workloads
        layers = int(sys.argv[2]) if len(sys.argv) > 2 else 13
        steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
        c4 = workloads()["C4"]
        wl = Workload("C4 layers", c4.layer_params[:layers], p=4, s=1, grad_dtype="bf16", hier_k=2, n=4)
        eng = Engine(n_ranks=4, arena_bytes=bench.arena_bytes(wl, 2, False, 4), devices=[0, 1])
        step = MicsStep(eng, wl, StepOptions(resident_grads=False))
        step.run(1)
        eng.synchronize()
        prof = step.profile()
        st = step.stats()
        t0 = time.perf_counter()
        step.run(steps)
        eng.synchronize()
        print(json.dumps({"op": "step (merged k_hier)", "layers": layers, "ms_per_step": (time.perf_counter() - t0) * 1e3
                          / steps, "allgather_ms": prof["allgather_ms"], "ag_launches": st.ag_launches,
                          "ag_nvlink_bytes_per_gpu": st.ag_remote_bytes,
                          "ag_nvlink_GBps": st.ag_remote_bytes / prof["allgather_ms"] / 1e6}), flush=True)
        step.close()
        eng.close()
        return
    from paper_2205_00119_b200.collectives import hierarchical_all_gather_device
    if mode == "peer":  # ncu-friendly: ONE GPU context (no cross-GPU kernel waits); ranks 2, 3's shards on GPU 1
        import ctypes as C
        chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 30_740_800 // 4 * 2
        reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
        cudart = C.CDLL("libcudart.so.12")
        for dev, peer in ((0, 1), (1, 0)):
            cudart.cudaSetDevice(dev)
            assert cudart.cudaDeviceEnablePeerAccess(peer, 0) in (0, 704)
        cudart.cudaSetDevice(0)
        eng = Engine(n_ranks=4, device=0, arena_bytes=6 * chunk + (256 << 20))
        src, out = eng.alloc(chunk), eng.alloc(4 * chunk)
        far = [torch.randint(0, 255, (chunk,), dtype=torch.uint8, device="cuda:1") for _ in range(2)]
        for r in range(2):
            eng.generate(src, r, chunk // 2, "bf16", seed=3, step=r)
        torch.cuda.synchronize(1)
        eng.synchronize()
        ptr_s = [eng.ptr(src, 0), eng.ptr(src, 1), far[0].data_ptr(), far[1].data_ptr()]
        ptr_o = [eng.ptr(out, r) for r in range(4)]
        ext = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", 0))
        run = lambda: hierarchical_all_gather_device(eng, 4, 2, ptr_s, chunk, ptr_o)  # noqa: E731
        run()
        eng.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(reps):
            run()
        e1.record(ext)
        eng.synchronize()
        ms = e0.elapsed_time(e1) / reps
        nvl = 2 * chunk  # ranks 0 and 1 each pull their channel peer's shard (ranks 2, 3) from GPU 1
        print(json.dumps({"op": "k_hier p=4 k=2, ranks 0-3 on GPU 0, shards of ranks 2-3 on GPU 1 (peer)",
                          "chunk_bytes": chunk, "ms": ms, "nvlink_bytes": nvl, "nvlink_GBps": nvl / ms / 1e6}),
              flush=True)
        eng.close()
        return
    chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 30_740_800 // 4 * 2
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
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
    ext = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(reps):
        run()
    e1.record(ext)
    eng.synchronize()
    ms = e0.elapsed_time(e1) / reps  # GPU 0's stream; the members meet at the launch's barriers
    nvl = 2 * (p // k - 1) * chunk   # per GPU per launch: 2 local ranks x (q-1) remote stage-1 chunks
    print(json.dumps({"op": "k_hier p=4 k=2 (one launch per call), 2 ranks/GPU on 2 GPUs", "chunk_bytes": chunk,
                      "ms": ms, "nvlink_bytes_per_gpu": nvl, "nvlink_GBps": nvl / ms / 1e6}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
