"""Collectives — the reference's API (collectives.hpp:64-112) over the sm_100a
pull engines.

Reference-shaped calls take host buffers (one per group position, numpy
arrays / bytes) and return fresh host buffers, exactly like the reference's
by-value ``std::vector<Bytes>`` API; they stage through the device (H2D,
kernel, D2H) and need a single-process engine.  The ``*_device`` variants take
device pointers (local or peer-mapped, from :meth:`Engine.ptr`) and only
enqueue work — they are the hot path and work across processes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import AgDesc, RsDesc, check, lib
from .engine import DTYPE_SIZE, NP_DTYPE, Engine, dtype_code
from .errors import Errc, raise_error
from .topology import ClusterSpec, GroupLayout

RS_STORE, RS_ACCUMULATE, RS_ZERO_ACCUM = 0, 1, 2


@dataclass
class CollectiveGroup:
    """collectives.hpp:30-36: ordered ranks; the position is the chunk index."""
    ranks: list = field(default_factory=list)

    def size(self) -> int:
        return len(self.ranks)

    def spans_nodes(self, cluster: ClusterSpec) -> bool:
        if not self.ranks:
            return False
        n0 = cluster.node_of(self.ranks[0])
        return any(cluster.node_of(r) != n0 for r in self.ranks)

    def validate(self) -> None:  # collectives.cpp:19-23
        if len(set(self.ranks)) != len(self.ranks):
            raise_error(Errc.ShapeError, "collective group has duplicate ranks")


def _ints(xs):
    return (C.c_int * max(len(xs), 1))(*xs)


def _ptrs(xs):
    return (C.c_void_p * max(len(xs), 1))(*[C.c_void_p(x) if x else None for x in xs])


def _bytes_of(buf) -> np.ndarray:
    if isinstance(buf, (bytes, bytearray)):
        return np.frombuffer(bytes(buf), np.uint8)
    return np.ascontiguousarray(buf).view(np.uint8).ravel()


def _check_equal_sizes(bufs, what):  # collectives.cpp:71-79
    for i in range(1, len(bufs)):
        if bufs[i].size != bufs[0].size:
            raise_error(Errc.SizeMismatch, f"{what}: buffer {i} has {bufs[i].size} bytes, expected {bufs[0].size}")


# ----------------------------------------------------------------------------- reference-shaped (host buffers)
def all_gather(engine: Engine, group: CollectiveGroup, shards) -> list:
    """collectives.cpp:103-134: every position gets C_0 || ... || C_{p-1}."""
    group.validate()
    p = group.size()
    if len(shards) != p:
        raise_error(Errc.SizeMismatch, f"all_gather: {len(shards)} shards for group of {p}")
    raw = [_bytes_of(s) for s in shards]
    _check_equal_sizes(raw, "all_gather")
    chunk = raw[0].size if raw else 0
    out = [np.empty(p * chunk, np.uint8) for _ in range(p)]
    check(lib.mics_host_all_gather(engine.ctx, _ints(group.ranks), p, _ptrs([r.ctypes.data for r in raw]), chunk,
                                   _ptrs([o.ctypes.data for o in out])))
    return out


def reduce_scatter(engine: Engine, group: CollectiveGroup, buffers, dtype: str) -> list:
    """collectives.cpp:136-183: position j gets fold_i buffers[i][chunk j], ascending position."""
    group.validate()
    p = group.size()
    if len(buffers) != p:
        raise_error(Errc.SizeMismatch, f"reduce_scatter: {len(buffers)} buffers for group of {p}")
    raw = [_bytes_of(b) for b in buffers]
    _check_equal_sizes(raw, "reduce_scatter")
    total = raw[0].size if raw else 0
    chunk = total // p if p else 0
    out = [np.empty(chunk, np.uint8) for _ in range(p)]
    check(lib.mics_host_reduce_scatter(engine.ctx, _ints(group.ranks), p, _ptrs([r.ctypes.data for r in raw]), total,
                                       dtype_code(dtype), _ptrs([o.ctypes.data for o in out])))
    return [o.view(NP_DTYPE[dtype]) for o in out]


def all_reduce(engine: Engine, group: CollectiveGroup, buffers, dtype: str) -> list:
    """collectives.cpp:185-190: reduce_scatter then all_gather."""
    group.validate()
    p = group.size()
    if len(buffers) != p:
        raise_error(Errc.SizeMismatch, f"reduce_scatter: {len(buffers)} buffers for group of {p}")
    raw = [_bytes_of(b) for b in buffers]
    _check_equal_sizes(raw, "reduce_scatter")
    total = raw[0].size if raw else 0
    out = [np.empty(total, np.uint8) for _ in range(p)]
    check(lib.mics_host_all_reduce(engine.ctx, _ints(group.ranks), p, _ptrs([r.ctypes.data for r in raw]), total,
                                   dtype_code(dtype), _ptrs([o.ctypes.data for o in out])))
    return [o.view(NP_DTYPE[dtype]) for o in out]


def hierarchical_all_gather(engine: Engine, layout: GroupLayout, cluster: ClusterSpec, shards,
                            corrupt_stage2: bool = False) -> list:
    """collectives.cpp:192-291: three-stage all-gather in every partition group;
    inputs/outputs indexed by global rank.  ``corrupt_stage2`` = HierarchicalOptions."""
    n = layout.n
    if cluster.total_ranks() != n:
        raise_error(Errc.ShapeError, f"cluster has {cluster.total_ranks()} ranks but layout expects {n}")
    if len(shards) != n:
        raise_error(Errc.SizeMismatch, f"hierarchical_all_gather: {len(shards)} shards for {n} ranks")
    raw = [_bytes_of(s) for s in shards]
    _check_equal_sizes(raw, "hierarchical_all_gather")
    chunk = raw[0].size if raw else 0
    out = [np.empty(layout.p * chunk, np.uint8) for _ in range(n)]
    check(lib.mics_host_hier_all_gather(engine.ctx, n, layout.p, cluster.devices_per_node,
                                        _ptrs([r.ctypes.data for r in raw]), chunk,
                                        _ptrs([o.ctypes.data for o in out]), int(corrupt_stage2)))
    return out


def batched_all_gather(engine: Engine, groups, shard_sets) -> list:
    """collectives.cpp:293-306: one coalesced launch for the whole batch."""
    if len(groups) != len(shard_sets):
        raise_error(Errc.SizeMismatch, f"batched_all_gather: {len(groups)} groups vs {len(shard_sets)} shard sets")
    sizes, ranks, chunks, srcs, outs, res = [], [], [], [], [], []
    for g, shards in zip(groups, shard_sets):
        g.validate()
        if len(shards) != g.size():
            raise_error(Errc.SizeMismatch, f"all_gather: {len(shards)} shards for group of {g.size()}")
        raw = [_bytes_of(s) for s in shards]
        _check_equal_sizes(raw, "all_gather")
        c = raw[0].size if raw else 0
        o = [np.empty(g.size() * c, np.uint8) for _ in range(g.size())]
        sizes.append(g.size())
        ranks += g.ranks
        chunks.append(c)
        srcs += [r.ctypes.data for r in raw]
        outs += [x.ctypes.data for x in o]
        res.append((o, raw))
    cnt = len(groups)
    check(lib.mics_host_batched_all_gather(engine.ctx, cnt, _ints(sizes), _ints(ranks),
                                           (C.c_uint64 * max(cnt, 1))(*chunks), _ptrs(srcs), _ptrs(outs)))
    return [o for o, _ in res]


def batched_reduce_scatter(engine: Engine, groups, buffer_sets, dtype: str) -> list:
    """collectives.cpp:308-321."""
    if len(groups) != len(buffer_sets):
        raise_error(Errc.SizeMismatch,
                    f"batched_reduce_scatter: {len(groups)} groups vs {len(buffer_sets)} buffer sets")
    sizes, ranks, nbytes, srcs, outs, res = [], [], [], [], [], []
    for g, bufs in zip(groups, buffer_sets):
        g.validate()
        if len(bufs) != g.size():
            raise_error(Errc.SizeMismatch, f"reduce_scatter: {len(bufs)} buffers for group of {g.size()}")
        raw = [_bytes_of(b) for b in bufs]
        _check_equal_sizes(raw, "reduce_scatter")
        total = raw[0].size if raw else 0
        o = [np.empty(total // g.size() if g.size() else 0, np.uint8) for _ in range(g.size())]
        sizes.append(g.size())
        ranks += g.ranks
        nbytes.append(total)
        srcs += [r.ctypes.data for r in raw]
        outs += [x.ctypes.data for x in o]
        res.append((o, raw))
    cnt = len(groups)
    check(lib.mics_host_batched_reduce_scatter(engine.ctx, cnt, _ints(sizes), _ints(ranks),
                                               (C.c_uint64 * max(cnt, 1))(*nbytes), _ptrs(srcs), dtype_code(dtype),
                                               _ptrs(outs)))
    return [[x.view(NP_DTYPE[dtype]) for x in o] for o, _ in res]


# ----------------------------------------------------------------------------- device pointers (hot path)
def all_gather_device(engine: Engine, ranks, shard_ptrs, chunk_bytes: int, out_ptrs) -> None:
    check(lib.mics_all_gather(engine.ctx, _ints(ranks), len(ranks), _ptrs(shard_ptrs), chunk_bytes, _ptrs(out_ptrs)))


def reduce_scatter_device(engine: Engine, ranks, in_ptrs, in_elems: int, out_ptrs, in_dtype: str = "f32",
                          acc_dtype: str | None = None, scale: float = 1.0, mode: int = RS_STORE,
                          valid_elems: int | None = None) -> None:
    acc = acc_dtype or ("f32" if in_dtype == "bf16" else in_dtype)
    check(lib.mics_reduce_scatter(engine.ctx, _ints(ranks), len(ranks), _ptrs(in_ptrs), in_elems,
                                  in_elems if valid_elems is None else valid_elems, dtype_code(in_dtype),
                                  dtype_code(acc), scale, mode, _ptrs(out_ptrs)))


def all_reduce_device(engine: Engine, ranks, buf_ptrs, elems: int, dtype: str = "f32") -> None:
    check(lib.mics_all_reduce(engine.ctx, _ints(ranks), len(ranks), _ptrs(buf_ptrs), elems, dtype_code(dtype)))


def hierarchical_all_gather_device(engine: Engine, p: int, k: int, shard_ptrs, chunk_bytes: int, out_ptrs,
                                   corrupt_stage2: bool = False) -> None:
    check(lib.mics_hier_all_gather(engine.ctx, p, k, _ptrs(shard_ptrs), chunk_bytes, _ptrs(out_ptrs),
                                   int(corrupt_stage2)))


def batched_all_gather_device(engine: Engine, descs) -> None:
    """descs: iterable of (ranks, shard_ptrs, chunk_bytes, out_ptrs)."""
    keep, arr = [], (AgDesc * max(len(descs), 1))()
    for i, (ranks, sp, cb, op) in enumerate(descs):
        r, s, o = _ints(ranks), _ptrs(sp), _ptrs(op)
        keep += [r, s, o]
        arr[i] = AgDesc(C.cast(r, C.POINTER(C.c_int)), len(ranks), C.cast(s, C.POINTER(C.c_void_p)), cb,
                        C.cast(o, C.POINTER(C.c_void_p)))
    check(lib.mics_batched_all_gather(engine.ctx, arr, len(descs)))


def batched_reduce_scatter_device(engine: Engine, descs, in_dtype: str = "f32", acc_dtype: str | None = None,
                                  scale: float = 1.0, mode: int = RS_STORE) -> None:
    """descs: iterable of (ranks, in_ptrs, in_elems, valid_elems, out_ptrs)."""
    acc = acc_dtype or ("f32" if in_dtype == "bf16" else in_dtype)
    keep, arr = [], (RsDesc * max(len(descs), 1))()
    for i, (ranks, ip, ne, nv, op) in enumerate(descs):
        r, s, o = _ints(ranks), _ptrs(ip), _ptrs(op)
        keep += [r, s, o]
        arr[i] = RsDesc(C.cast(r, C.POINTER(C.c_int)), len(ranks), C.cast(s, C.POINTER(C.c_void_p)), ne, nv,
                        C.cast(o, C.POINTER(C.c_void_p)))
    check(lib.mics_batched_reduce_scatter(engine.ctx, arr, len(descs), dtype_code(in_dtype), dtype_code(acc), scale,
                                          mode))


class Plan:
    """A persistent collective (descriptor table uploaded once; ``run`` replays it)."""

    def __init__(self, engine: Engine, handle):
        self.engine = engine
        self.h = handle

    def run(self, iterations: int = 1) -> None:
        check(lib.mics_plan_run(self.engine.ctx, self.h, iterations))

    def close(self) -> None:
        if self.h:
            check(lib.mics_plan_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def plan_all_gather(engine: Engine, ranks, shard_ptrs, chunk_bytes: int, out_ptrs) -> Plan:
    h = C.c_void_p()
    check(lib.mics_plan_all_gather(engine.ctx, _ints(ranks), len(ranks), _ptrs(shard_ptrs), chunk_bytes,
                                   _ptrs(out_ptrs), C.byref(h)))
    return Plan(engine, h)


def plan_reduce_scatter(engine: Engine, ranks, in_ptrs, in_elems: int, out_ptrs, in_dtype: str = "f32",
                        acc_dtype: str | None = None, scale: float = 1.0, mode: int = RS_STORE,
                        valid_elems: int | None = None) -> Plan:
    acc = acc_dtype or ("f32" if in_dtype == "bf16" else in_dtype)
    h = C.c_void_p()
    check(lib.mics_plan_reduce_scatter(engine.ctx, _ints(ranks), len(ranks), _ptrs(in_ptrs), in_elems,
                                       in_elems if valid_elems is None else valid_elems, dtype_code(in_dtype),
                                       dtype_code(acc), scale, mode, _ptrs(out_ptrs), C.byref(h)))
    return Plan(engine, h)


__all__ = ["Plan", "plan_all_gather", "plan_reduce_scatter","CollectiveGroup", "all_gather", "reduce_scatter", "all_reduce", "hierarchical_all_gather",
           "batched_all_gather", "batched_reduce_scatter", "all_gather_device", "reduce_scatter_device",
           "all_reduce_device", "hierarchical_all_gather_device", "batched_all_gather_device",
           "batched_reduce_scatter_device", "RS_STORE", "RS_ACCUMULATE", "RS_ZERO_ACCUM", "DTYPE_SIZE"]
