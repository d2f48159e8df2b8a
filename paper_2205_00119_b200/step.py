"""MiCS step driver (host side of csrc/step.cpp) and the BASELINE.json workloads.

A step = s micro-steps of {per-layer parameter all-gather (fwd), per-layer
all-gather (bwd), coalesced gradient reduce-scatter} + the boundary all-reduce
fused with sharded fp32 Adam (simulator.cpp:265-280 order, executed for real).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from ._lib import Buf, StepCfg, StepStats, check, lib
from .engine import DTYPE, Engine
from .workloads import Workload, workloads  # noqa: F401  (re-exported: the step's workload description)


@dataclass
class StepOptions:
    resident_grads: bool = True
    alternative: bool = False     # DeepSpeed-default global all-reduce every micro-step instead of 2-hop
    seed: int = 2205
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    compute: bool = False         # layer GEMMs in the step (tcgen05, K7); gradients come from them
    recompute: bool = False       # recompute Y_l in the backward pass instead of storing it


class MicsStep:
    def __init__(self, engine: Engine, wl: Workload, opts: StepOptions = field(default_factory=StepOptions)):
        if not isinstance(opts, StepOptions):
            opts = StepOptions()
        self.engine = engine
        self.wl = wl
        self.opts = opts
        self._layers = (C.c_uint64 * len(wl.layer_params))(*wl.layer_params)
        cfg = StepCfg(wl.p, wl.s, len(wl.layer_params), C.cast(self._layers, C.POINTER(C.c_uint64)),
                      DTYPE[wl.grad_dtype], wl.hier_k, int(opts.resident_grads), int(opts.alternative), opts.seed,
                      opts.lr, opts.beta1,
                      opts.beta2, opts.eps, opts.weight_decay, int(opts.compute), int(opts.recompute),
                      wl.tokens if opts.compute else 0, wl.hidden if opts.compute else 0)
        h = C.c_void_p()
        check(lib.mics_step_create(engine.ctx, C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            check(lib.mics_step_destroy(self.h))
            self.h = None

    def run(self, iterations: int = 1) -> None:
        """Enqueue `iterations` global steps on the engine's stream."""
        check(lib.mics_step_run(self.engine.ctx, self.h, iterations))

    def run_host(self, host_grads_ptr: int, iterations: int = 1, host_result_ptr: int | None = None) -> None:
        check(lib.mics_step_run_host(self.engine.ctx, self.h, C.c_void_p(host_grads_ptr), iterations,
                                     C.c_void_p(host_result_ptr) if host_result_ptr else None))

    def profile(self) -> dict:
        """One serialised step with CUDA events around every phase (ms)."""
        ms = (C.c_double * 5)()
        check(lib.mics_step_profile_ex(self.engine.ctx, self.h, ms))
        return {"allgather_ms": ms[0], "reducescatter_ms": ms[1], "boundary_ms": ms[2], "generate_ms": ms[3],
                "gemm_ms": ms[4]}

    def stats(self) -> StepStats:
        s = StepStats()
        check(lib.mics_step_stats_get(self.h, C.byref(s)))
        return s

    def buffers(self) -> dict:
        bufs = [Buf() for _ in range(6)]
        check(lib.mics_step_buffers(self.h, *[C.byref(b) for b in bufs]))
        return dict(zip(["param_bf16", "master", "exp_avg", "exp_avg_sq", "gathered", "grads"], bufs))

    def sync_info(self):
        from ._lib import SyncInfo
        h = C.c_void_p()
        check(lib.mics_step_sync(self.h, C.byref(h)))
        info = SyncInfo()
        check(lib.mics_sync_get_info(h, C.byref(info)))
        segs = []
        for i in range(info.nseg):
            ln, ch, so, go = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            check(lib.mics_sync_seg(h, i, C.byref(ln), C.byref(ch), C.byref(so), C.byref(go)))
            segs.append((ln.value, ch.value, so.value, go.value))
        return info, segs
