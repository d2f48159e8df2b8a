"""2-hop gradient synchronisation — the reference's sync_schedule.hpp API over
device-resident sync states.

``make_sync_states`` returns a :class:`SyncStates` handle (the reference returns
``std::vector<SyncState<T>>``); the shards live on the GPU.  The schedule calls
mirror the reference (two_hop_micro_step :118-147, two_hop_boundary :153-185,
alternative_schedule_step :189-224, alternative_boundary :228-232) including the
``BoundaryViolation`` state machine (:87-103) and the optional SyncEvent log.
Gradients are host arrays (one per rank, length grad_len) for the drop-in calls,
or a symmetric device buffer for the hot path (:meth:`SyncStates.micro_step_device`).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from ._lib import Adam, Buf, SyncInfo, check, lib
from .engine import DTYPE_SIZE, NP_DTYPE, Engine, dtype_code
from .errors import Errc, raise_error
from .topology import GroupLayout

RS_STORE, RS_ACCUMULATE, RS_ZERO_ACCUM = 0, 1, 2


class SyncPhase(enum.IntEnum):  # sync_schedule.hpp:14
    micro_rs = 0
    boundary_ar = 1
    global_ar = 2


def phase_name(p: SyncPhase) -> str:
    return SyncPhase(p).name


@dataclass(frozen=True)
class SyncEvent:  # sync_schedule.hpp:27-32
    step: int
    phase: SyncPhase
    group_id: int
    bytes: int


def owned_chunk_elems(layout: GroupLayout, grad_len: int) -> int:  # :53-56
    return (grad_len + layout.p - 1) // layout.p


@dataclass
class AdamConfig:
    """Sharded fp32 Adam fused into the boundary all-reduce (not in the reference)."""
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    step: int = 1
    grad_scale: float = 1.0
    write_grad: bool = False


class SyncStates:
    """SyncState<T> of every rank (sync_schedule.hpp:45-51), shards on the device."""

    def __init__(self, engine: Engine, layout: GroupLayout, seg_lens, s: int, dtype: str = "f32",
                 align_elems: int = 1):
        if layout.n != engine.n:
            raise_error(Errc.ShapeError, f"layout has {layout.n} ranks but the engine has {engine.n}")
        self.engine = engine
        self.layout = layout
        self.dtype = dtype
        self._mark0 = engine.mark()  # arena is a bump allocator: close() pops our allocations if on top
        lens = (C.c_uint64 * len(seg_lens))(*seg_lens)
        h = C.c_void_p()
        check(lib.mics_sync_create(engine.ctx, layout.p, s, len(seg_lens), lens, dtype_code(dtype), align_elems,
                                   C.byref(h)))
        self.h = h
        info = self.info()
        self.s = info.s
        self.shard_elems = info.shard_elems
        self.grad_elems = info.grad_elems
        self.segs = []
        for i in range(len(seg_lens)):
            ln, ch, so, go = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            check(lib.mics_sync_seg(self.h, i, C.byref(ln), C.byref(ch), C.byref(so), C.byref(go)))
            self.segs.append((ln.value, ch.value, so.value, go.value))
        self._grads = {}  # dtype -> staging Buf for the host drop-in calls
        self._mark1 = engine.mark()

    def _track(self, top_before: int):
        """Calls may allocate lazily (staging, scratch, flags).  Our allocations stay
        poppable only while nobody else allocated on top of them."""
        if top_before == self._mark1:
            self._mark1 = self.engine.mark()
        else:
            self._mark1 = -1  # interleaved with foreign allocations: never pop

    def close(self):
        if getattr(self, "h", None):
            check(lib.mics_sync_destroy(self.h))
            self.h = None
            if self.engine.ctx and self.engine.mark() == self._mark1:
                self.engine.release(self._mark0)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def info(self) -> SyncInfo:
        i = SyncInfo()
        check(lib.mics_sync_get_info(self.h, C.byref(i)))
        return i

    @property
    def micro_step(self) -> int:
        return self.info().micro_step

    @property
    def shard_buf(self) -> Buf:
        return self.info().shard

    def shard(self, rank: int) -> np.ndarray:
        """The rank's accumulated owned shard (host copy)."""
        return self.engine.d2h(self.shard_buf, rank, self.shard_elems, self.dtype)

    def shards(self) -> list:
        return [self.shard(r) for r in self.engine.local_ranks]

    # ---- hot path: gradients already on the device (padded segment layout)
    def micro_step_device(self, grads: Buf, grad_dtype: str | None = None, off: int = 0, scale: float = 1.0,
                          mode: int = RS_ACCUMULATE) -> None:
        check(lib.mics_sync_micro_step(self.engine.ctx, self.h, grads, off, dtype_code(grad_dtype or self.dtype),
                                       scale, mode))

    def alt_step_device(self, grads: Buf, grad_dtype: str | None = None, off: int = 0, scale: float = 1.0) -> None:
        top = self.engine.mark()
        check(lib.mics_sync_alt_step(self.engine.ctx, self.h, grads, off, dtype_code(grad_dtype or self.dtype), scale))
        self._track(top)

    def boundary(self, adam: Adam | None = None) -> None:
        top = self.engine.mark()
        check(lib.mics_sync_boundary(self.engine.ctx, self.h, C.byref(adam) if adam is not None else None))
        self._track(top)

    def alt_boundary(self) -> None:
        check(lib.mics_sync_alt_boundary(self.engine.ctx, self.h))

    def events(self) -> list:
        cnt = C.c_uint64(0)
        check(lib.mics_sync_events(self.h, None, 0, C.byref(cnt)))
        buf = (C.c_int64 * (4 * max(cnt.value, 1)))()
        check(lib.mics_sync_events(self.h, buf, cnt.value, C.byref(cnt)))
        return [SyncEvent(buf[4 * i], SyncPhase(buf[4 * i + 1]), buf[4 * i + 2], buf[4 * i + 3])
                for i in range(cnt.value)]

    def clear_events(self) -> None:
        check(lib.mics_sync_clear_events(self.h))

    # ---- drop-in: stage host gradients into the padded device layout
    def stage_grads(self, grads, dtype: str | None = None) -> Buf:
        dtype = dtype or self.dtype
        if dtype not in self._grads:
            top = self.engine.mark()
            self._grads[dtype] = self.engine.alloc(self.grad_elems * DTYPE_SIZE[dtype])
            self._track(top)
        buf = self._grads[dtype]
        if len(grads) != self.layout.n:
            raise_error(Errc.SizeMismatch, "gradient count does not match rank count")
        for r in self.engine.local_ranks:
            g = np.ascontiguousarray(grads[r], NP_DTYPE[dtype]).ravel()
            pos = 0
            for ln, ch, _, go in self.segs:
                piece = g[pos:pos + ln]
                pos += ln
                if piece.size:
                    self.engine.h2d(buf, r, piece, off=go * DTYPE_SIZE[dtype])
        return buf


def make_sync_states(engine: Engine, layout: GroupLayout, grad_len: int, s: int, dtype: str = "f32") -> SyncStates:
    """make_sync_states<T> (:58-69): shards of ceil(len/p) zeros, micro_step 0."""
    if s < 1:
        raise_error(Errc.OutOfRange, "micro-step count s must be >= 1")
    return SyncStates(engine, layout, [grad_len], s, dtype)


def _log(states: SyncStates, log, before: int):
    if log is not None:
        log.extend(states.events()[before:])


def two_hop_micro_step(engine: Engine, layout: GroupLayout, states: SyncStates, grads, log=None) -> None:
    """:118-147 — reduce-scatter inside every partition group, shard += result."""
    before = len(states.events()) if log is not None else 0
    if states.micro_step >= states.s:  # check before staging, like the reference (:123)
        raise_error(Errc.BoundaryViolation, f"micro-step past accumulation boundary (micro_step = s = {states.s})")
    buf = states.stage_grads(grads)
    states.micro_step_device(buf, mode=RS_ACCUMULATE)
    _log(states, log, before)


def two_hop_boundary(engine: Engine, layout: GroupLayout, states: SyncStates, log=None,
                     adam: Adam | None = None) -> None:
    """:153-185 — all-reduce inside every replication group (optionally fused with Adam)."""
    before = len(states.events()) if log is not None else 0
    states.boundary(adam)
    _log(states, log, before)


def alternative_schedule_step(engine: Engine, layout: GroupLayout, states: SyncStates, grads, log=None) -> None:
    """:189-224 — all-reduce across all n ranks every micro-step; keep the owned chunk."""
    before = len(states.events()) if log is not None else 0
    if states.micro_step >= states.s:
        raise_error(Errc.BoundaryViolation, f"micro-step past accumulation boundary (micro_step = s = {states.s})")
    buf = states.stage_grads(grads)
    states.alt_step_device(buf)
    _log(states, log, before)


def alternative_boundary(states: SyncStates) -> None:
    """:228-232."""
    states.alt_boundary()


def make_adam(states: SyncStates, cfg: AdamConfig, param: Buf, exp_avg: Buf, exp_avg_sq: Buf,
              param_bf16: Buf | None = None) -> Adam:
    return Adam(cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, cfg.step, cfg.grad_scale, param, exp_avg,
                exp_avg_sq, param_bf16 if param_bf16 is not None else Buf(0, 0), int(cfg.write_grad))
