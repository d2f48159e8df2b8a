"""MiCS step benchmark (BASELINE.json metric: MiCS step samples/s at 1/2/4/8 B200;
partition-group collective GB/s vs NVLink).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl mics|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)
  python bench.py --sweep ...                              (C2: AG/RS sweep 1 MiB..1 GiB vs NCCL)

A step is one global MiCS step of the workload: s micro-steps of {per-layer bf16
parameter all-gather fwd + bwd, coalesced fp32/bf16 gradient reduce-scatter} and the
boundary replication-group all-reduce fused with sharded fp32 Adam.  The job has
n = 8 ranks (the configs' 8 ranks) laid out node-major over the N GPUs, n/N virtual
ranks per GPU: at N=1 every collective is intra-GPU (HBM-bound), at N=8 every
partition group spans GPUs (NVLink-bound).  Total work is fixed ("strong").
samples/s = n * micro_batch(8) * s / step time.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_RANKS = 8
MICRO_BATCH = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--impl", default="mics", choices=["mics", "reference"])
    ap.add_argument("--ranks", type=int, default=N_RANKS)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--generated-grads", action="store_true", help="generate gradients inside the step (K6)")
    ap.add_argument("--schedule", default="two_hop", choices=["two_hop", "alternative"],
                    help="2-hop sync (MiCS) or the DeepSpeed-default all-reduce over all ranks every micro-step")
    ap.add_argument("--p", type=int, default=0, help="override the workload's partition group size (ablation)")
    ap.add_argument("--micro-steps", type=int, default=0, help="override s, micro-steps per step (ablation)")
    ap.add_argument("--sweep", action="store_true", help="C2 collective sweep instead of the step")
    ap.add_argument("--compute", action="store_true",
                    help="headline = the step with its layer GEMMs (tcgen05), gathers overlapped with compute")
    ap.add_argument("--no-compute", action="store_true", help="skip the step-with-compute sub-measurement")
    ap.add_argument("--compute-steps", type=int, default=3)
    ap.add_argument("--no-collectives", action="store_true",
                    help="skip the per-N partition-group collective GB/s points (N > 1)")
    return ap.parse_args()


def env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-lms", "100"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def bind_to_gpu_numa(local):
    """Pin this process to the CPUs of the GPU's own NUMA node (sysfs local_cpulist)
    so the pinned host buffers of the e2e path are allocated next to its PCIe root
    (MICS_NUMA=0 disables).  Returns the CPU list used, or None."""
    if os.environ.get("MICS_NUMA") == "0":
        return None
    try:
        import torch
        pr = torch.cuda.get_device_properties(local)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as fh:
            spec = fh.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return spec
    except (OSError, AttributeError, ValueError):
        return None
    return None



def arena_bytes(wl, per, resident, n=N_RANKS, alternative=False, compute=None):
    """Per-process arena for `per` local ranks (mirrors csrc/step.cpp's allocations).
    compute: None (communication step) or "store" / "recompute" (step with compute)."""
    p, s = wl.p, wl.s
    chunks = [((e + p - 1) // p + 7) // 8 * 8 for e in wl.layer_params]
    S = sum(chunks)
    r = n // p
    sub = ((S + r - 1) // r + 3) // 4 * 4
    szg = 2 if wl.grad_dtype == "bf16" else 4
    hmerge = wl.hier_k and p > wl.hier_k and os.environ.get("MICS_HIER_MERGE") != "0"  # merged hierarchical launches
    slots_ag = (2 if compute else 3 * int(os.environ.get("MICS_HIER_VISITS", "3")) if hmerge
                else max(3, min(8, int(os.environ.get("MICS_GATHER_SLOTS", "3")))))  # csrc/step.cpp
    gathered = slots_ag * (((max(chunks) * p * 2) + 255) // 256 * 256)
    slots = min(2, s) if compute else (s if resident else 1)
    per_rank = r * sub * 4 + S * 2 + 3 * S * 4 + gathered + slots * p * S * szg
    if wl.hier_k and p > wl.hier_k:  # stage-1 tile flags of the hierarchical gathers
        per_rank += slots_ag * (p // wl.hier_k) * (-(-max(chunks) * 2 // 32768)) * 8 + 4096
    if compute:
        T, h = wl.tokens, wl.hidden
        ldy = [(e // h + 7) // 8 * 8 for e in wl.layer_params]
        per_rank += s * T * h * 2 + T * h * 4 + T * (max(ldy) if compute == "recompute" else sum(ldy)) * 2
        if per < p:  # partition groups span GPUs: copy-engine staging of the peers' chunks (csrc/step.cpp ce_rs)
            per_rank += p * S * szg
    if alternative:  # all-n reduce-scatter scratch: n slices of ceil(p*chunk/n) per layer
        per_rank += sum(-(-p * c // n) * n for c in chunks) * 4
    return per * (per_rank + 8 * 4096) + (256 << 20)


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=GLOO)
    return float(t.item())


GLOO = None


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier(group=GLOO)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def ncu_traffic(workload, n_gpus, phase):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel,
    from the committed `ncu --set full` captures (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            table = json.load(fh)
    except OSError:
        return None
    ent = table.get(f"{workload.split(' ')[0]}|{n_gpus}|{phase}")
    return ent["dram_bytes_per_launch"] if ent else None


# ----------------------------------------------------------------------------- config (both arms)
def grad_elems(wl):
    """Padded gradient elements per rank (csrc/step.cpp: chunk = ceil(E/p) rounded to 8)."""
    return sum(((e + wl.p - 1) // wl.p + 7) // 8 * 8 * wl.p for e in wl.layer_params)


def config_for(wl, args, world):
    """The workload description both arms print (the driver compares them key by key):
    pure function of the workload and the command line."""
    szg = 2 if wl.grad_dtype == "bf16" else 4
    n = args.ranks
    return {"workload": wl.name, "n_ranks": n, "ranks_per_gpu": n // world, "p": wl.p, "s": wl.s,
            "micro_batch": MICRO_BATCH, "params": wl.params, "grad_dtype": wl.grad_dtype,
            "param_dtype": "bf16 (fp32 master, m, v)", "hierarchical_k": wl.hier_k,
            "l2": "inputs larger than L2 (gradient sets of %.2f GB/rank)" % (wl.s * grad_elems(wl) * szg / 1e9),
            "parallelism": f"MiCS p={wl.p} x {n // wl.p} replicas", "schedule": args.schedule}


# ----------------------------------------------------------------------------- CPU baseline (reference)
def ref_layer_seconds(wl, threads, size, port=None):
    """Wall seconds of the reference's own step functions (oracle/_ref, compiled from
    the unmodified sources) over ONE layer of `size` parameters for all n ranks:
    per-layer all_gather fwd + bwd in every partition group, two_hop_micro_step x s,
    two_hop_boundary, plus the Adam loop the reference lacks (oracle/ref_shim.cpp
    ref_step_sample).  Falls back to the plain-C restatement (`port`) when the
    reference was not built.  Returns (seconds, kind, threads used)."""
    import ctypes as C
    from oracle.oracle import REF_SO, RefLib
    if RefLib.available():
        lib = C.CDLL(REF_SO)
        lib.ref_step_sample.restype = C.c_double
        arr = (C.c_uint64 * 1)(size)
        return lib.ref_step_sample(threads, wl.n, wl.p, wl.s, 1, arr, 1), "reference", threads
    import numpy as np
    from oracle.oracle import Oracle
    ora = port or Oracle()
    n, p, s, ln = wl.n, wl.p, wl.s, size
    g = np.random.default_rng(0).standard_normal((s, n, ln)).astype(np.float32)
    sh = np.zeros((p, (ln + p - 1) // p * 2), np.uint8)
    t0 = time.perf_counter()
    for _ in range(s):
        for _ in range(2 * n // p):
            ora.all_gather(sh)
    out, _, _ = ora.two_hop(g, n, p, "f32")
    for r in range(n):
        ora.adam(np.zeros(out.shape[1]), np.zeros(out.shape[1]), np.zeros(out.shape[1]), out[r], 1e-4, 0.9,
                 0.999, 1e-8, 0.0, 1, 1.0 / (n * s))
    return time.perf_counter() - t0, "port", 1


def layer_sizes(wl):
    """{size: count} over the workload's layers; the most frequent size is the per-step sample."""
    sizes = {}
    for e in wl.layer_params:
        sizes[e] = sizes.get(e, 0) + 1
    block = max(sizes, key=lambda e: (sizes[e], e))
    return sizes, block


def cpu_baseline(wl, threads, calib=None):
    """The reference's CPU step for the whole model, assembled from per-layer timings:
    every distinct layer size is timed once at full size (C3: the 31.8M-parameter
    embedding and one 12.6M-parameter block, all 8 ranks), and the step time is the
    sum over the model's layers — the reference's step cost is a sum of independent
    per-layer collectives plus element-wise 2-hop / Adam work."""
    sizes, block = layer_sizes(wl)
    t = dict(calib or {})
    kind = "reference"
    for e in sizes:
        if e not in t:
            t[e], kind, threads = ref_layer_seconds(wl, threads, e)
    if any(v <= 0 for v in t.values()):
        return None
    step_s = sum(t[e] * c for e, c in sizes.items())
    timed = ", ".join(f"{c} x {e:,}-param layer at {t[e]:.2f} s" for e, c in sizes.items())
    return {"value": N_RANKS * MICRO_BATCH * wl.s / step_s, "unit": "samples/s", "cores": threads, "kind": kind,
            "sample": f"each distinct layer size timed once at full size (all {wl.n} ranks, p={wl.p}, s={wl.s}: "
                      f"per-layer all_gather fwd+bwd, two_hop_micro_step x s, two_hop_boundary, Adam loop); "
                      f"step = {timed} = {step_s:.1f} s (sum over layers)",
            "step_seconds": step_s, "extrapolated": len(wl.layer_params) > len(sizes), "layer_seconds": t}


def run_reference(args, wl, rank, world):
    """`--impl reference`: the reference's own CPU implementation (oracle/_ref: the
    unmodified sdpsim sources) on the box's host cores, same workload and config.
    The full C3 step takes ~70 s on 16 cores, so each timed step is a bounded sample:
    one full-size transformer block for all 8 ranks (the other layer sizes are
    timed once up front); `value` is the whole-model step assembled from them
    (`extrapolated`), `ms_per_step` the sample actually timed per step."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sizes, block = layer_sizes(wl)
    calib = {}
    for e in sizes:
        if e != block:
            calib[e], kind, threads = ref_layer_seconds(wl, threads, e)
    samples = []
    for i in range(args.warmup + args.steps):
        sec, kind, threads = ref_layer_seconds(wl, threads, block)
        if sec <= 0:
            print(json.dumps({"impl": "reference", "unavailable": "reference step sample failed"}))
            return
        if i >= args.warmup:
            samples.append(sec)
    t_block = statistics.median(samples)
    cb = cpu_baseline(wl, threads, calib | {block: t_block})
    v = cb["value"]
    line = {"impl": "reference", "metric": "MiCS step samples/s", "value": v, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * t_block, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "config": config_for(wl, args, world),
            "extrapolated": True,
            "extrapolation": {"timed_per_step": f"one {block:,}-parameter layer, all {wl.n} ranks",
                              "sample_ms_per_step": 1000 * t_block,
                              "full_step_ms": 1000 * cb["step_seconds"],
                              "other_layers_timed_once_s": calib,
                              "formula": "step = sum over layers of the timed per-layer seconds; "
                                         "value = n * micro_batch * s / step"},
            "cpu_baseline": {"kind": cb["kind"], "cores": cb["cores"], "sample": cb["sample"], "value": v,
                             "unit": "samples/s"},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- NCCL comparator
def graph_or_eager(fn, warmup):
    """The comparator's step captured once in a CUDA graph and replayed (no per-call
    host launch cost inside the timed region, like libmics' graph-replayed step);
    `warmup` eager calls on a side stream first.  Falls back to eager calls if the
    capture is refused.  Returns (callable, "cuda_graph" | "eager")."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(max(1, warmup)):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g.replay, "cuda_graph"
    except Exception:  # noqa: BLE001
        torch.cuda.synchronize()
        return fn, "eager"


def nccl_step(wl, rank, world, steps, warmup):
    """The same MiCS step with stock NCCL collectives on split communicators and
    torch's fused Adam (only meaningful with one rank per GPU), graph-captured."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    p, s, n = wl.p, wl.s, world
    pg = {g: dist.new_group(list(range(g * p, (g + 1) * p))) for g in range(n // p)}
    rg = {j: dist.new_group(list(range(j, n, p))) for j in range(p)}
    my_pg, my_rg = pg[rank // p], rg[rank % p]
    chunks = [((e + p - 1) // p + 7) // 8 * 8 for e in wl.layer_params]
    S = sum(chunks)
    gdt = torch.bfloat16 if wl.grad_dtype == "bf16" else torch.float32
    shard = torch.randn(S, device=dev).to(torch.bfloat16)
    gathered = torch.empty(2 * max(chunks) * p, dtype=torch.bfloat16, device=dev)
    grads = [torch.randn(p * S, device=dev).to(gdt) for _ in range(s)]
    acc = torch.zeros(S, dtype=torch.float32, device=dev)
    tmp = torch.empty(S, dtype=gdt, device=dev)
    master = torch.nn.Parameter(torch.randn(S, device=dev))
    opt = torch.optim.Adam([master], lr=1e-4, fused=True, capturable=True)
    master.grad = acc
    offs = [0]
    for c in chunks:
        offs.append(offs[-1] + c)

    def one():
        for t in range(s):
            for order in (range(len(chunks)), reversed(range(len(chunks)))):
                for l in order:
                    c = chunks[l]
                    out = gathered[(l % 2) * max(chunks) * p:(l % 2) * max(chunks) * p + c * p]
                    dist.all_gather_into_tensor(out, shard[offs[l]:offs[l] + c], group=my_pg)
            dist.reduce_scatter_tensor(tmp, grads[t], group=my_pg)
            acc.add_(tmp.float()) if t else acc.copy_(tmp.float())
        if n // p > 1:
            dist.all_reduce(acc, group=my_rg)
        opt.step()
        shard.copy_(master.detach().to(torch.bfloat16))

    run, mode = graph_or_eager(one, warmup)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    e1.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    return {"value": n * MICRO_BATCH * s / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "launch": mode,
            "what": "torch.distributed NCCL all_gather_into_tensor / reduce_scatter_tensor / all_reduce on split "
                    "groups + torch.optim.Adam(fused, capturable), same shapes, one CUDA graph per step"}


def nccl_compute_step(wl, rank, world, steps, warmup):
    """Comparator for the step with compute, one rank per GPU: the same model and
    schedule on the stock stack — torch.matmul (cuBLAS) for the layer GEMMs, NCCL
    all_gather_into_tensor on a side stream one layer ahead (prefetch), NCCL
    reduce_scatter_tensor per micro-step, all_reduce at the boundary, fused Adam.
    Timing only (random data).  Like the K7 path it pads every layer's row count to
    a multiple of 8: cuBLAS on the unpadded, 2-byte-misaligned shapes (12301 rows)
    ran at 130-160 TF/s (tools/probe_stock.py)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    p, s, n, T, h = wl.p, wl.s, world, wl.tokens, wl.hidden
    pg = {g: dist.new_group(list(range(g * p, (g + 1) * p))) for g in range(n // p)}
    rg = {j: dist.new_group(list(range(j, n, p))) for j in range(p)}
    my_pg, my_rg = pg[rank // p], rg[rank % p]
    ldy = [(e // h + 7) // 8 * 8 for e in wl.layer_params]
    # per layer: a gradient region of R_l (>= the padded dW, divisible by p) and a shard of R_l / p
    R = [(max(((e + p - 1) // p + 7) // 8 * 8 * p, r * h) + p - 1) // p * p for e, r in zip(wl.layer_params, ldy)]
    offs, goffs = [0], [0]
    for r_ in R:
        offs.append(offs[-1] + r_ // p)
        goffs.append(goffs[-1] + r_)
    S, G = offs[-1], goffs[-1]
    gdt = torch.bfloat16 if wl.grad_dtype == "bf16" else torch.float32
    shard = (torch.randn(S, device=dev) * 0.02).to(torch.bfloat16)
    gathered = [torch.zeros(max(R), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    X = [torch.randn(T, h, device=dev).to(torch.bfloat16) for _ in range(s)]
    Y = [torch.empty(T, r, dtype=torch.bfloat16, device=dev) for r in ldy]
    dX = torch.zeros(T, h, dtype=torch.float32, device=dev)
    grads = [torch.zeros(G, dtype=gdt, device=dev) for _ in range(2)]
    acc = torch.zeros(S, dtype=torch.float32, device=dev)
    tmp = torch.empty(S, dtype=gdt, device=dev)
    master = torch.nn.Parameter(shard.float())
    opt = torch.optim.Adam([master], lr=1e-4, fused=True, capturable=True)
    master.grad = acc
    side = torch.cuda.Stream()
    ev_g = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    L = len(ldy)

    def gather(l):
        b = l % 2
        with torch.cuda.stream(side):
            side.wait_event(ev_free[b])
            dist.all_gather_into_tensor(gathered[b][:R[l]], shard[offs[l]:offs[l + 1]], group=my_pg)
            ev_g[b].record(side)

    def W(l):
        return gathered[l % 2][:ldy[l] * h].view(ldy[l], h)

    def one():
        main = torch.cuda.current_stream()  # a capture stream when graph-captured
        side.wait_stream(main)  # the side stream joins this stream's work (and a capture)
        for e in ev_free:
            e.record(main)
        for t in range(s):
            g = grads[t % 2]
            gather(0)
            for l in range(L):  # forward, prefetching layer l+1
                if l + 1 < L:
                    gather(l + 1)
                main.wait_event(ev_g[l % 2])
                torch.matmul(X[t], W(l).t(), out=Y[l])
                ev_free[l % 2].record(main)
            gather(L - 1)
            for l in range(L - 1, -1, -1):  # backward
                if l > 0:
                    gather(l - 1)
                main.wait_event(ev_g[l % 2])
                Wl = W(l)
                if l == L - 1:  # bf16 cuBLAS products, accumulated / stored in the step's dtypes
                    dX.copy_(torch.matmul(Y[l], Wl))
                else:
                    dX.add_(torch.matmul(Y[l], Wl))
                dW = g[goffs[l]:goffs[l] + ldy[l] * h].view(ldy[l], h)
                if gdt == torch.bfloat16:
                    torch.matmul(Y[l].t(), X[t], out=dW)
                else:
                    dW.copy_(torch.matmul(Y[l].t(), X[t]))
                ev_free[l % 2].record(main)
            dist.reduce_scatter_tensor(tmp, g, group=my_pg)
            acc.add_(tmp.float()) if t else acc.copy_(tmp.float())
        if n // p > 1:
            dist.all_reduce(acc, group=my_rg)
        opt.step()
        shard.copy_(master.detach().to(torch.bfloat16))
        main.wait_stream(side)  # rejoin the side stream

    def timed(run):
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            run()
        e1.record()
        e1.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / steps, world)

    # both launch modes, the faster one reported: graph capture removes host launch
    # cost, but measured slower here (the captured NCCL kernels overlap the GEMMs less)
    run, mode = graph_or_eager(one, warmup)
    times = {mode: timed(run)}
    if mode != "eager":
        times["eager"] = timed(one)
    mode = min(times, key=times.get)
    ms = times[mode]
    return {"value": n * MICRO_BATCH * s / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "launch": mode,
            "ms_per_step_by_launch": times,
            "what": "same model and schedule on torch.matmul (cuBLAS, rows padded to 8) + NCCL all_gather (side "
                    "stream, one layer ahead) / reduce_scatter / all_reduce + torch.optim.Adam(fused=True)"}


# ----------------------------------------------------------------------------- step with compute
def measure_compute(args, wl, rank, world, local):
    """The MiCS step with its layer GEMMs (tcgen05, K7): gradients come from the GEMMs,
    gathers prefetch on their own stream under the GEMMs (SURVEY §8f items 2+3).
    Returns the measurement dict (rank 0's view, times max over ranks)."""
    import torch

    from paper_2205_00119_b200 import dist as mdist
    from paper_2205_00119_b200.engine import Engine, host_alloc, host_free
    from paper_2205_00119_b200.step import MicsStep, StepOptions

    n = args.ranks
    per = n // world
    free = torch.cuda.mem_get_info(local)[0]
    mode = "store"
    if arena_bytes(wl, per, False, n, compute="store") > 0.92 * free:
        mode = "recompute"  # activations do not fit: recompute Y_l in the backward pass
    need = arena_bytes(wl, per, False, n, compute=mode)
    if need > 0.95 * free:
        return {"error": f"{per} ranks/GPU need {need / 1e9:.1f} GB, {free / 1e9:.1f} GB free"}
    eng = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=need)
    mdist.connect(eng, GLOO)
    step = MicsStep(eng, wl, StepOptions(compute=True, recompute=mode == "recompute"))
    stats = step.stats()
    ext = torch.cuda.ExternalStream(eng.stream())
    steps = max(2, args.compute_steps)
    step.run(args.warmup)
    eng.synchronize()
    barrier(world)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    l0 = eng.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.barrier()
    eng.synchronize()
    barrier(world)
    e0.record(ext)
    step.run(steps)
    e1.record(ext)
    e1.synchronize()
    eng.synchronize()
    barrier(world)
    clk = clocks.stop()
    launches = (eng.launches - l0) // steps
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    prof = step.profile()  # serialised: every phase timed alone
    prof = {k: max_over_ranks(v, world) for k, v in prof.items()}
    serial_ms = sum(prof[k] for k in ("allgather_ms", "reducescatter_ms", "boundary_ms", "gemm_ms"))
    comm_ms = serial_ms - prof["gemm_ms"]
    pk, pk_kind = peaks()
    tf_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    gemm_tflops = stats.compute_flops / (prof["gemm_ms"] / 1e3) / 1e12 if prof["gemm_ms"] > 0 else 0.0
    samples = n * MICRO_BATCH * wl.s
    out = {"value": samples / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "steps": steps,
           "activations": mode, "tokens_per_micro_batch": wl.tokens, "hidden": wl.hidden,
           "model": "parallel-branch linear proxy: layer l = its parameters as W_l [E_l/hidden, hidden], "
                    "loss 1/2 sum_l ||X W_l^T||^2 (fwd Y=XW^T, bwd dX+=YW, dW=Y^T X; no attention/norms)",
           "tflop_per_step_per_gpu": stats.compute_flops / 1e12,
           "achieved_tflops_per_gpu": stats.compute_flops / (ms / 1e3) / 1e12,
           "serialised_phases_ms": prof, "serialised_ms": serial_ms,
           "overlap": {"comm_ms": comm_ms, "gemm_ms": prof["gemm_ms"],
                       "hidden_comm_frac": max(0.0, min(1.0, (serial_ms - ms) / comm_ms)) if comm_ms > 0 else None},
           "roofline": {"bound": "tensor", "kernel": "k_gemm (tcgen05 bf16, K7)", "achieved": gemm_tflops,
                        "peak": tf_peak, "unit": "TFLOP/s", "frac": gemm_tflops / tf_peak,
                        "peak_source": f"MEASURED_PEAKS.json bf16_tflops_sustained ({pk_kind}; kernel inside a long "
                                       "step)", "traffic": None,
                        "launch_ms": prof["gemm_ms"] / max(1, stats.gemm_launches),
                        "launches_per_step": stats.gemm_launches},
           "gpu_launches": launches * steps, "clocks": clk}
    if not args.no_e2e and args.e2e_steps > 0:
        xb = wl.tokens * wl.hidden * 2
        host, hptr = host_alloc(xb)
        import numpy as np
        host[:] = np.random.default_rng(rank).integers(0x3c00, 0x3f80, xb // 2, dtype=np.uint16).view(np.uint8)
        res, rptr = host_alloc(per * 4096 * 4)
        step.run_host(hptr, 1, rptr)
        eng.synchronize()
        barrier(world)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        h0.record(ext)
        step.run_host(hptr, args.e2e_steps, rptr)
        h1.record(ext)
        h1.synchronize()
        wall = (time.perf_counter() - t0) / args.e2e_steps
        ems = max_over_ranks(max(h0.elapsed_time(h1) / args.e2e_steps, wall * 1e3), world)
        out["e2e"] = {"value": samples / (ems / 1e3), "unit": "samples/s", "ms_per_step": ems,
                      "h2d_bytes_per_step": per * wl.s * xb, "d2h_bytes_per_step": per * 4096 * 4,
                      "path": "mics_step_run_host (C-ABI): pinned host inputs X (tokens x hidden bf16) -> H2D every "
                              "micro-step and rank, updated master slice D2H after the boundary"}
        host_free(hptr)
        host_free(rptr)
    step.close()
    eng.close()
    if world > 1 and per == 1:
        try:
            out["nccl_cublas_comparator"] = nccl_compute_step(wl, rank, world, max(2, args.compute_steps), 1)
        except Exception as e:  # noqa: BLE001
            out["nccl_cublas_comparator"] = {"error": str(e)[:200]}
    return out


# ----------------------------------------------------------------------------- main arm
def run_mics(args, wl, rank, world, local):
    import torch

    from paper_2205_00119_b200 import dist as mdist
    from paper_2205_00119_b200.step import MicsStep, StepOptions
    from paper_2205_00119_b200.engine import Engine, host_alloc, host_free

    torch.cuda.set_device(local)
    numa = bind_to_gpu_numa(local)
    n = args.ranks
    if n % world:
        raise SystemExit(f"--gpus {world} must divide the {n} ranks")
    per = n // world
    resident = not args.generated_grads
    alt = args.schedule == "alternative"
    free = torch.cuda.mem_get_info(local)[0]

    def need(res):
        return arena_bytes(wl, per, res, n, alt)
    if resident and need(True) > 0.92 * free:
        resident = False  # s resident gradient sets do not fit (C5): generate them per micro-step (K6)
    if need(resident) > 0.95 * free:
        raise SystemExit(f"{wl.name}: {per} ranks/GPU need {need(resident) / 1e9:.1f} GB, "
                         f"{free / 1e9:.1f} GB free — use more GPUs")
    eng = Engine(n_ranks=n, world=world, world_rank=rank, device=local, arena_bytes=need(resident))
    mdist.connect(eng, GLOO)
    step = MicsStep(eng, wl, StepOptions(resident_grads=resident, alternative=args.schedule == "alternative"))
    stats = step.stats()
    ext = torch.cuda.ExternalStream(eng.stream())

    # warm-up, then the timed region (barrier + sync on both sides)
    step.run(args.warmup)
    eng.synchronize()
    barrier(world)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    l0 = eng.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.barrier()
    eng.synchronize()
    barrier(world)
    e0.record(ext)
    step.run(args.steps)
    e1.record(ext)
    e1.synchronize()
    eng.synchronize()
    barrier(world)
    clk = clocks.stop()
    launches = eng.launches - l0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    samples = n * MICRO_BATCH * wl.s
    value = samples / (ms / 1e3)

    # per-phase device times (CUDA events on the launching stream), one extra step
    prof = step.profile()
    prof = {k: max_over_ranks(v, world) for k, v in prof.items()}
    # algorithmic bytes per phase, summed by the library from the planned descriptor
    # tables (this process, per step): pulled from peers over NVLink / local HBM r+w
    kernels = {"allgather": "k_copy (per-layer partition-group all-gather)",
               "reducescatter": "k_reduce (micro-step reduce-scatter + shard accumulate)",
               "boundary": ("k_tail (K8: last micro-step reduce-scatter + boundary all-reduce + Adam, one pass)"
                            if world == 1 else
                            "k_fbnd (K9: per layer group boundary all-reduce + Adam in one launch, block flags)"
                            if wl.n // wl.p > 1 else "k_adam (shards already reduced: Adam only)")}
    phases = {"allgather": (prof["allgather_ms"], stats.ag_launches, stats.ag_remote_bytes, stats.ag_hbm_bytes),
              "reducescatter": (prof["reducescatter_ms"], stats.rs_launches, stats.rs_remote_bytes,
                                stats.rs_hbm_bytes),
              "boundary": (prof["boundary_ms"], stats.bnd_launches, stats.bnd_remote_bytes, stats.bnd_hbm_bytes)}
    dom = max(phases, key=lambda k: phases[k][0])
    dom_ms, dom_launches, remote, hbm = phases[dom]
    dom_launches = max(1, dom_launches)
    pk, pk_kind = peaks()
    per_launch_s = dom_ms / dom_launches / 1e3
    nv_gbs = remote / dom_launches / per_launch_s / 1e9
    hbm_gbs = hbm / dom_launches / per_launch_s / 1e9
    if remote and remote / NVLINK_PEER_GBS >= hbm / pk["hbm_gbs"]:  # the resource with the longer ideal time
        roof = {"bound": "nvlink", "achieved": nv_gbs, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": nv_gbs / NVLINK_PEER_GBS,
                "peak_source": "measured peer copy 770 GB/s per direction (B200_PROFILING.md; 900 nominal). "
                               "Both directions loaded at once (every GPU sends and receives): 670 GB/s pull, "
                               "706 GB/s push measured by tools/probe_bulk.cu",
                "bytes_per_launch": remote / dom_launches}
    else:
        roof = {"bound": "hbm", "achieved": hbm_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_gbs / pk["hbm_gbs"], "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})",
                "bytes_per_launch": hbm / dom_launches}
    roof.update({"traffic": ncu_traffic(wl.name, world, dom), "kernel": kernels[dom], "phase": dom,
                 "launch_ms": per_launch_s * 1e3, "launches_per_step": dom_launches, "nvlink_GBps": nv_gbs,
                 "hbm_GBps": hbm_gbs})
    p, s = wl.p, wl.s
    S = stats.shard_elems
    szg = 2 if wl.grad_dtype == "bf16" else 4

    # end-to-end through the C-ABI with host buffers: gradients H2D every micro-step
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        gbytes = stats.grad_elems * szg
        host, hptr = host_alloc(gbytes)  # one gradient set, copied for every local rank and micro-step
        res, rptr = host_alloc(per * 4096 * 4)
        import numpy as np
        pat = np.random.default_rng(rank).standard_normal(1 << 22).astype(
            np.float32 if szg == 4 else np.float32).view(np.uint8)
        if szg == 2:
            pat = pat.view(np.uint32).astype(np.uint32).view(np.uint16)[1::2].copy().view(np.uint8)
        for o in range(0, host.size, pat.size):  # synthetic gradient values, tiled
            host[o:o + pat.size] = pat[:host.size - o]
        step.run_host(hptr, 1, rptr)  # warm-up
        eng.synchronize()
        barrier(world)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        h0.record(ext)
        step.run_host(hptr, args.e2e_steps, rptr)
        h1.record(ext)
        h1.synchronize()
        wall = (time.perf_counter() - t0) / args.e2e_steps
        ems = max_over_ranks(max(h0.elapsed_time(h1) / args.e2e_steps, wall * 1e3), world)
        e2e = {"value": samples / (ems / 1e3), "unit": "samples/s", "ms_per_step": ems,
               "h2d_bytes_per_step": per * s * gbytes, "d2h_bytes_per_step": per * min(4096, S) * 4,
               "h2d_GBps_per_gpu": per * s * gbytes / (ems / 1e3) / 1e9,
               "bound": "host link: every rank's fp32 gradients of every micro-step cross PCIe (the reference API "
                        "takes host gradients); h2d_GBps_per_gpu is the achieved host->GPU rate",
               "path": "mics_step_run_host (C-ABI): pinned host gradients -> H2D every micro-step, "
                       "result slice D2H after the boundary",
               "host_cpus": numa}
        host_free(hptr)
        host_free(rptr)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, os.cpu_count() or 1)
        if cpu and cpu["kind"] == "reference" and (os.cpu_count() or 1) > 1:
            # the reference's engine at 1 thread too (the block only, scaled by
            # the nproc run's per-layer ratio to keep the bench within minutes)
            sizes, block = layer_sizes(wl)
            t1, _, _ = ref_layer_seconds(wl, 1, block)
            if t1 > 0:
                step1 = cpu["step_seconds"] * t1 / cpu["layer_seconds"][block]
                cpu["single_thread"] = {"value": N_RANKS * MICRO_BATCH * wl.s / step1, "cores": 1,
                                        "step_seconds": step1, "block_seconds": t1}

    nccl = None
    if world > 1 and per == 1:
        try:
            nccl = nccl_step(wl, rank, world, max(2, args.steps // 2), 1)
        except Exception as e:  # noqa: BLE001
            nccl = {"error": str(e)[:200]}

    line = {
        "metric": "MiCS step samples/s", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_for(wl, args, world),
        "run": {"grads": "resident in HBM (generated before timing)" if resident else "generated in-step (K6)",
                "launch": "stream" if os.environ.get("MICS_GRAPH") == "0"
                          else "CUDA graph replay (one graph per step)"},
        "roofline": roof,
        "phases_ms": {k: v[0] for k, v in phases.items()},
        "per_rank_bytes": {"allgather_in": stats.ag_bytes_in, "reducescatter_in": stats.rs_bytes_in,
                           "boundary_in": stats.ar_bytes_in, "adam_hbm": stats.adam_hbm_bytes},
        "phase_GBps": {k: {"nvlink": v[2] / (v[0] / 1e3) / 1e9, "hbm": v[3] / (v[0] / 1e3) / 1e9}
                       for k, v in phases.items() if v[0] > 0},
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "nccl_comparator": nccl,
    }
    step.close()
    eng.close()
    if world > 1 and not args.no_collectives:
        # partition-group collectives vs NVLink at this GPU count (BASELINE.json metric, second
        # half): one rank per GPU, p in {2, 4, 8} dividing N, 256 MiB and 1 GiB, libmics vs NCCL
        try:
            from tools.sweep import run_sweep
            pts = run_sweep(args, rank, world, local, sizes=[256 << 20, 1 << 30], quiet=True)
            line["collectives"] = [{"op": r["op"], "p": r["p"], "bytes": r["bytes"],
                                    "busbw_GBps": round(r["mics_busbw_GBps"], 1),
                                    "frac_of_770": round(r["frac_nvlink_770"], 3),
                                    "nccl_busbw_GBps": round(r["nccl_busbw_GBps"], 1) if r["nccl_busbw_GBps"] else None}
                                   for r in pts]
            big = [r for r in pts if r["bytes"] >= (1 << 30)]
            line["collectives_summary"] = {
                "points": len(pts),
                "beats_nccl": sum(1 for r in pts if r["nccl_us"] and r["mics_us"] < r["nccl_us"]),
                "min_frac_of_770_at_1GiB": round(min(r["frac_nvlink_770"] for r in big), 3) if big else None,
                "p": sorted({r["p"] for r in pts})}
        except Exception as e:  # noqa: BLE001
            line["collectives"] = {"error": str(e)[:200]}
    if not args.no_compute and wl.hidden and args.schedule == "two_hop":
        try:
            line["compute_step"] = measure_compute(args, wl, rank, world, local)
        except Exception as e:  # noqa: BLE001  (the headline stays the communication step)
            line["compute_step"] = {"error": str(e)[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_compute_headline(args, wl, rank, world, local):
    """`--compute`: the step with its layer GEMMs as the headline line."""
    c = measure_compute(args, wl, rank, world, local)
    if "error" in c:
        raise SystemExit(c["error"])
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, os.cpu_count() or 1)
    line = {"metric": "MiCS step samples/s (with layer GEMMs)", "value": c["value"], "unit": "samples/s",
            "n_gpus": world, "steps": c["steps"], "warmup": args.warmup, "ms_per_step": c["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16 GEMMs, f32 sync",
            "data": "synthetic",
            "config": {"workload": wl.name + " + layer GEMMs", "n_ranks": args.ranks, "ranks_per_gpu":
                       args.ranks // world, "p": wl.p, "s": wl.s, "micro_batch": MICRO_BATCH,
                       "tokens_per_micro_batch": wl.tokens, "hidden": wl.hidden, "params": wl.params,
                       "grad_dtype": wl.grad_dtype, "activations": c["activations"],
                       "l2": "inputs larger than L2", "launch": "CUDA graph replay (gathers / GEMMs / sync streams)"},
            "roofline": c["roofline"], "e2e": c.get("e2e"), "gpu_launches": c["gpu_launches"],
            "clocks": c["clocks"], "cpu_baseline": cpu,
            "nccl_cublas_comparator": c.get("nccl_cublas_comparator"),
            "detail": {k: c[k] for k in ("model", "tflop_per_step_per_gpu", "achieved_tflops_per_gpu",
                                         "serialised_phases_ms", "serialised_ms", "overlap")}}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    global GLOO
    args = parse()
    rank, world, local = env()
    # pure Python: the reference arm never loads libmics (the package __init__ is lazy)
    from paper_2205_00119_b200.workloads import workloads
    wl = workloads()[args.workload]
    if args.p or args.micro_steps:
        import dataclasses
        wl = dataclasses.replace(wl, p=args.p or wl.p, s=args.micro_steps or wl.s)
        wl.name = re.sub(r"p=\d+", f"p={wl.p}", re.sub(r"s=\d+", f"s={wl.s}", wl.name))
        if wl.p != wl.n:
            wl.name = wl.name.replace(" (ZeRO-3)", "")
        if f"p={wl.p}" not in wl.name:
            wl.name += f", p={wl.p}"
        if f"s={wl.s}" not in wl.name:
            wl.name += f", s={wl.s}"
    if args.impl == "reference":  # CPU only: no process group, ranks > 0 exit without work
        run_reference(args, wl, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group(backend="cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
        GLOO = dist.new_group(backend="gloo")
    if args.sweep:
        from tools.sweep import run_sweep
        run_sweep(args, rank, world, local)
    elif args.compute:
        run_compute_headline(args, wl, rank, world, local)
    else:
        run_mics(args, wl, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier(group=GLOO)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
