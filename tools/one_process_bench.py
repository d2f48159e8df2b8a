"""The MiCS step with one process driving several GPUs (mics_init_devices) — the
reference's single in-process engine over NVLink — timed like bench.py: W warm-up
steps, K timed steps between CUDA events recorded on EVERY member's stream, the max
over members.  Compare with `torchrun --nproc-per-node N bench.py --gpus N`.

    python tools/one_process_bench.py [--gpus N] [--workload C3] [--steps K] [--warmup W]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions
    from paper_2205_00119_b200.workloads import workloads
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    wl, n, N = workloads()[a.workload], 8, a.gpus
    per = n // N
    free = min(torch.cuda.mem_get_info(d)[0] for d in range(N))
    resident = bench.arena_bytes(wl, per, True, n) <= 0.92 * free
    eng = Engine(n_ranks=n, arena_bytes=bench.arena_bytes(wl, per, resident, n), devices=list(range(N)))
    step = MicsStep(eng, wl, StepOptions(resident_grads=resident))
    step.run(a.warmup)
    eng.synchronize()
    ev = []
    for d in range(N):
        s = torch.cuda.ExternalStream(eng.device_stream(d), device=torch.device("cuda", d))
        with torch.cuda.device(d):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev.append((s, e0, e1))
    for s, e0, _ in ev:
        e0.record(s)
    step.run(a.steps)
    for s, _, e1 in ev:
        e1.record(s)
    eng.synchronize()
    ms = max(e0.elapsed_time(e1) for _, e0, e1 in ev) / a.steps
    print(json.dumps({"metric": "MiCS step samples/s (one process, mics_init_devices)", "workload": wl.name,
                      "gpus": N, "ranks_per_gpu": per, "ms_per_step": ms,
                      "value": n * bench.MICRO_BATCH * wl.s / (ms / 1e3), "grads": "resident" if resident else
                      "generated in-step"}), flush=True)
    step.close()
    eng.close()


if __name__ == "__main__":
    main()
