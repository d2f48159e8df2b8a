"""The engine: B200 counterpart of the reference's ``VirtualRankEngine``
(collectives.hpp:42-62, collectives.cpp:25-67).

An :class:`Engine` owns one ``mics_ctx``: n virtual ranks laid out node-major
over ``world`` processes (one per GPU), a symmetric device arena, a CUDA
stream and the per-(sender, receiver) traffic log the reference keeps.
``num_threads`` is the engine's worker count, as in the reference: here the CTAs
per SM every collective runs with (``None`` = one resident wave at each kernel's
occupancy; ``set_parallelism`` also caps CTAs per launch).  Results and traffic
never depend on it — the reference's contract (collectives.hpp:38-41), pinned by
tests/test_gpu_determinism.py.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import IPC_HANDLE_BYTES, Buf, InitArgs, check, lib

DTYPE = {"i64": 0, "f32": 1, "f64": 2, "bf16": 3}
NP_DTYPE = {"i64": np.int64, "f32": np.float32, "f64": np.float64, "bf16": np.uint16, "u8": np.uint8}
DTYPE_SIZE = {"i64": 8, "f32": 4, "f64": 8, "bf16": 2}


def dtype_code(dtype) -> int:
    if isinstance(dtype, str):
        return DTYPE[dtype]
    return int(dtype)


class Engine:
    def __init__(self, num_threads: int | None = None, *, n_ranks: int = 64, world: int = 1, world_rank: int = 0,
                 device: int = 0, arena_bytes: int = 1 << 30, devices=None):
        """One GPU (`device`), one GPU of a `world`-process job, or — `devices` — one
        process driving several GPUs (mics_init_devices): ranks node-major over them,
        `arena_bytes` per GPU."""
        self.num_threads = None if num_threads is None else max(1, int(num_threads))
        self.n = n_ranks
        self.world = world
        self.world_rank = world_rank
        self.devices = list(devices) if devices else [device]
        self.device = self.devices[0]
        args = InitArgs(n_ranks, world, world_rank, self.device, arena_bytes)
        ctx = C.c_void_p()
        if devices:
            arr = (C.c_int * len(self.devices))(*self.devices)
            check(lib.mics_init_devices(C.byref(args), arr, len(self.devices), C.byref(ctx)))
        else:
            check(lib.mics_init(C.byref(args), C.byref(ctx)))
        self.ctx = ctx
        first, count = C.c_int(0), C.c_int(0)
        check(lib.mics_local_ranks(self.ctx, C.byref(first), C.byref(count)))
        self.local_ranks = list(range(first.value, first.value + count.value))
        if self.num_threads is not None:
            self.set_parallelism(self.num_threads)

    def set_parallelism(self, ctas_per_sm: int = 0, max_ctas: int = 0) -> None:
        """Worker CTAs per SM (0 = occupancy) and per launch (0 = no cap) of every
        collective planned from now on (mics_set_parallelism)."""
        check(lib.mics_set_parallelism(self.ctx, int(ctas_per_sm), int(max_ctas)))

    # ------------------------------------------------------------ lifetime
    def close(self) -> None:
        if getattr(self, "ctx", None):
            check(lib.mics_destroy(self.ctx))
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    # ------------------------------------------------------------ multi-process plumbing
    def export_handle(self) -> bytes:
        buf = (C.c_char * IPC_HANDLE_BYTES)()
        check(lib.mics_ipc_export(self.ctx, buf))
        return bytes(buf)

    def import_handles(self, handles: list) -> None:
        blob = b"".join(handles)
        assert len(blob) == IPC_HANDLE_BYTES * self.world
        cbuf = C.create_string_buffer(blob, len(blob))
        check(lib.mics_ipc_import(self.ctx, cbuf))

    def gpu_of(self, rank: int) -> int:
        """The CUDA device hosting `rank` (multi-device contexts: node-major placement)."""
        return self.devices[rank // (self.n // len(self.devices))] if len(self.devices) > 1 else self.device

    def process_of(self, rank: int) -> int:
        out = C.c_int(0)
        check(lib.mics_rank_process(self.ctx, rank, C.byref(out)))
        return out.value

    def is_local(self, rank: int) -> bool:
        return rank in self.local_ranks

    # ------------------------------------------------------------ memory
    def alloc(self, bytes_per_rank: int) -> Buf:
        b = Buf()
        check(lib.mics_alloc(self.ctx, int(bytes_per_rank), C.byref(b)))
        return b

    def mark(self) -> int:
        m = C.c_uint64(0)
        check(lib.mics_arena_mark(self.ctx, C.byref(m)))
        return m.value

    def release(self, mark: int) -> None:
        check(lib.mics_arena_release(self.ctx, mark))

    def arena_used(self):
        u, c = C.c_uint64(0), C.c_uint64(0)
        check(lib.mics_arena_used(self.ctx, C.byref(u), C.byref(c)))
        return u.value, c.value

    def ptr(self, buf: Buf, rank: int) -> int:
        out = C.c_void_p()
        check(lib.mics_buf_ptr(self.ctx, buf, rank, C.byref(out)))
        return out.value

    def h2d(self, buf: Buf, rank: int, array: np.ndarray, off: int = 0) -> None:
        a = np.ascontiguousarray(array)
        check(lib.mics_h2d(self.ctx, buf, rank, off, a.ctypes.data_as(C.c_void_p), a.nbytes))
        self.synchronize()  # `a` may be a temporary

    def d2h(self, buf: Buf, rank: int, count: int, dtype: str = "f32", off: int = 0) -> np.ndarray:
        out = np.empty(count, NP_DTYPE[dtype])
        check(lib.mics_d2h(self.ctx, buf, rank, off, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def memset(self, buf: Buf, rank: int, nbytes: int, value: int = 0, off: int = 0) -> None:
        check(lib.mics_memset(self.ctx, buf, rank, off, value, nbytes))

    def generate(self, buf: Buf, rank: int, count: int, dtype: str = "f32", seed: int = 0, step: int = 0,
                 layer: int = 0, start: int = 0, off: int = 0) -> None:
        """K6: counter-based synthetic values (splitmix64), same formula as oracle/mics_oracle.c."""
        check(lib.mics_generate(self.ctx, buf, rank, off, dtype_code(dtype), seed, step, layer, start, count))

    # ------------------------------------------------------------ execution
    def stream(self) -> int:
        s = C.c_void_p()
        check(lib.mics_stream(self.ctx, C.byref(s)))
        return s.value or 0

    def device_stream(self, d: int) -> int:
        """cudaStream_t of member d of a multi-device context (d = 0 otherwise)."""
        out = C.c_void_p()
        check(lib.mics_device_stream(self.ctx, d, C.byref(out)))
        return out.value

    def synchronize(self) -> None:
        check(lib.mics_synchronize(self.ctx))

    def barrier(self) -> None:
        check(lib.mics_barrier(self.ctx))

    @property
    def launches(self) -> int:
        out = C.c_uint64(0)
        check(lib.mics_launch_count(self.ctx, C.byref(out)))
        return out.value

    @property
    def num_sms(self) -> int:
        out = C.c_int(0)
        check(lib.mics_num_sms(self.ctx, C.byref(out)))
        return out.value

    # ------------------------------------------------------------ traffic log (collectives.cpp:46-67)
    def traffic(self) -> dict:
        n = C.c_uint64(0)
        check(lib.mics_traffic_size(self.ctx, C.byref(n)))
        buf = (C.c_int64 * (3 * max(n.value, 1)))()
        check(lib.mics_traffic_get(self.ctx, buf, n.value))
        return {(buf[3 * i], buf[3 * i + 1]): buf[3 * i + 2] for i in range(n.value)}

    def bytes_received_by(self, rank: int) -> int:
        return sum(b for (_, to), b in self.traffic().items() if to == rank)

    def clear_traffic(self) -> None:
        check(lib.mics_traffic_clear(self.ctx))

    def enable_traffic(self, on: bool = True) -> None:
        check(lib.mics_traffic_enable(self.ctx, int(on)))


def host_alloc(nbytes: int):
    """Pinned host memory (cudaHostAlloc) as a numpy uint8 array + its raw pointer."""
    p = C.c_void_p()
    check(lib.mics_host_alloc(nbytes, C.byref(p)))
    arr = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value))
    return arr, p.value


def host_free(ptr: int) -> None:
    check(lib.mics_host_free(C.c_void_p(ptr)))
