"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end of the CPU checker.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(``paper_2205_00119_b200``) never does.

Two checkers live behind it:

* ``Oracle``  — ``oracle/liboracle.so``, the plain-C restatement
  (``oracle/mics_oracle.c``).  Always buildable (``make -C oracle``).
* ``RefLib``  — ``oracle/_ref/libsdpsim_ref.so``, the unmodified reference hot
  path (``/root/reference/proj/src/{topology,collectives}.cpp`` +
  ``sync_schedule.hpp``) behind ``oracle/ref_shim.cpp``.  Built only where
  ``/root/reference`` exists (``make -C oracle ref``); travels to the GPU box
  as a prebuilt file and is optional everywhere.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsdpsim_ref.so")

DTYPES = {"i64": 0, "f32": 1, "f64": 2}
NP = {"i64": np.int64, "f32": np.float32, "f64": np.float64}

_P = C.c_void_p
_I = C.c_int
_SZ = C.c_size_t


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_oracle(force: bool = False) -> None:
    if force or not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)


def build_ref() -> bool:
    """Compile the reference into oracle/_ref when /root/reference exists."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(REF_SO)
    subprocess.check_call(["make", "-s", "-C", HERE, "ref"], stdout=subprocess.DEVNULL,
                          stderr=subprocess.DEVNULL)
    return True


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle status {code}: {what}")
        self.code = code


class Oracle:
    """The plain-C restatement."""

    def __init__(self):
        build_oracle()
        self.lib = C.CDLL(ORACLE_SO)
        L = self.lib
        L.ora_splitmix64.restype = C.c_uint64
        L.ora_splitmix64.argtypes = [C.c_uint64]
        L.ora_f32_to_bf16.restype = C.c_uint16
        L.ora_f32_to_bf16.argtypes = [C.c_float]

    def f32_to_bf16(self, a):
        """Round-to-nearest-even bf16 of every element (ora_f32_to_bf16)."""
        a = np.ascontiguousarray(a, np.float32).ravel()
        return np.array([self.lib.ora_f32_to_bf16(float(x)) for x in a], np.uint16)

    # ---- generators
    def random_shards(self, count, chunk, seed):
        out = np.empty(count * chunk, np.uint8)
        self.lib.ora_mt_random_shards(_I(count), _SZ(chunk), C.c_uint32(seed), _ptr(out))
        return out.reshape(count, chunk)

    def random_i64(self, count, lo, hi, seed):
        out = np.empty(count, np.int64)
        self.lib.ora_mt_random_i64(_SZ(count), C.c_int64(lo), C.c_int64(hi), C.c_uint32(seed), _ptr(out))
        return out

    def random_f32(self, count, lo, hi, seed):
        out = np.empty(count, np.float32)
        self.lib.ora_mt_random_f32(_SZ(count), C.c_float(lo), C.c_float(hi), C.c_uint32(seed), _ptr(out))
        return out

    def gen_f32(self, seed, rank, step, layer, start, count):
        out = np.empty(count, np.float32)
        self.lib.ora_gen_f32(C.c_uint64(seed), _I(rank), _I(step), _I(layer), C.c_uint64(start), _SZ(count),
                             _ptr(out))
        return out

    def gen_bf16(self, seed, rank, step, layer, start, count):
        out = np.empty(count, np.uint16)
        self.lib.ora_gen_bf16(C.c_uint64(seed), _I(rank), _I(step), _I(layer), C.c_uint64(start), _SZ(count),
                              _ptr(out))
        return out

    # ---- topology
    def build_group_layout(self, n, p):
        part = np.zeros(max(n, 1), np.int32)
        repl = np.zeros(max(n, 1), np.int32)
        st = self.lib.ora_build_group_layout(_I(n), _I(p), _ptr(part), _ptr(repl))
        if st:
            raise OracleError(st)
        return part.reshape(n // p, p), repl.reshape(p, n // p)

    def partition_shape_ok(self, p, k):
        return bool(self.lib.ora_partition_shape_ok(_I(p), _I(k)))

    def min_feasible_partition(self, states, num_nodes, k, device_memory, node_granular, headroom=0.85):
        out = C.c_int(0)
        st = self.lib.ora_min_feasible_partition(C.c_uint64(states), _I(num_nodes), _I(k), C.c_uint64(device_memory),
                                                 _I(int(node_granular)), C.c_double(headroom), C.byref(out))
        if st:
            raise OracleError(st)
        return out.value

    # ---- collectives (arrays indexed by group position)
    def all_gather(self, shards: np.ndarray) -> np.ndarray:
        shards = np.ascontiguousarray(shards, np.uint8)
        p, chunk = shards.shape
        out = np.empty((p, p * chunk), np.uint8)
        self.lib.ora_all_gather(_I(p), _ptr(shards), _SZ(chunk), _ptr(out))
        return out

    def reduce_scatter(self, bufs: np.ndarray, dtype: str) -> np.ndarray:
        bufs = np.ascontiguousarray(bufs)
        p = bufs.shape[0]
        raw = bufs.view(np.uint8).reshape(p, -1)
        nbytes = raw.shape[1]
        out = np.empty((p, nbytes // max(p, 1)), np.uint8)
        st = self.lib.ora_reduce_scatter(_I(p), _ptr(raw), _SZ(nbytes), _I(DTYPES[dtype]), _ptr(out))
        if st:
            raise OracleError(st)
        return out.view(NP[dtype])

    def all_reduce(self, bufs: np.ndarray, dtype: str) -> np.ndarray:
        bufs = np.ascontiguousarray(bufs)
        p = bufs.shape[0]
        raw = bufs.view(np.uint8).reshape(p, -1)
        out = np.empty_like(raw)
        st = self.lib.ora_all_reduce(_I(p), _ptr(raw), _SZ(raw.shape[1]), _I(DTYPES[dtype]), _ptr(out))
        if st:
            raise OracleError(st)
        return out.view(NP[dtype])

    def hier_all_gather(self, shards: np.ndarray, p: int, k: int, corrupt: bool = False) -> np.ndarray:
        shards = np.ascontiguousarray(shards, np.uint8)
        n, chunk = shards.shape
        out = np.empty((n, p * chunk), np.uint8)
        st = self.lib.ora_hier_all_gather(_I(n), _I(p), _I(k), _ptr(shards), _SZ(chunk), _I(int(corrupt)), _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def traffic_all_gather(self, ranks, chunk, n, mat=None):
        mat = np.zeros((n, n), np.uint64) if mat is None else mat
        r = np.asarray(ranks, np.int32)
        self.lib.ora_traffic_all_gather(_ptr(r), _I(len(r)), _SZ(chunk), _I(n), _ptr(mat))
        return mat

    def traffic_reduce_scatter(self, ranks, nbytes, n, mat=None):
        mat = np.zeros((n, n), np.uint64) if mat is None else mat
        r = np.asarray(ranks, np.int32)
        self.lib.ora_traffic_reduce_scatter(_ptr(r), _I(len(r)), _SZ(nbytes), _I(n), _ptr(mat))
        return mat

    def traffic_all_reduce(self, ranks, nbytes, n, mat=None):
        mat = np.zeros((n, n), np.uint64) if mat is None else mat
        r = np.asarray(ranks, np.int32)
        self.lib.ora_traffic_all_reduce(_ptr(r), _I(len(r)), _SZ(nbytes), _I(n), _ptr(mat))
        return mat

    def traffic_hier_all_gather(self, n, p, k, chunk, corrupt=False):
        mat = np.zeros((n, n), np.uint64)
        st = self.lib.ora_traffic_hier_all_gather(_I(n), _I(p), _I(k), _SZ(chunk), _I(int(corrupt)), _ptr(mat))
        if st:
            raise OracleError(st)
        return mat

    # ---- schedules; grads: (s, n, len)
    def _sched(self, fn, grads, n, p, dtype, with_traffic=False):
        grads = np.ascontiguousarray(grads, NP[dtype])
        s, n_, length = grads.shape
        assert n_ == n
        chunk = (length + p - 1) // p
        out = np.zeros((n, chunk), NP[dtype])
        ev = np.zeros((4 * (s * n + n + 8), 1), np.int64).ravel()
        nev = C.c_int(0)
        traffic = np.zeros((n, n), np.uint64) if with_traffic else None
        st = fn(_I(DTYPES[dtype]), _I(n), _I(p), _I(s), _SZ(length), _ptr(grads), _ptr(out), _ptr(ev),
                _I(len(ev) // 4), C.byref(nev), _ptr(traffic))
        if st:
            raise OracleError(st)
        events = ev[: 4 * nev.value].reshape(-1, 4)
        return out, events, traffic

    def two_hop(self, grads, n, p, dtype, with_traffic=False):
        return self._sched(self.lib.ora_two_hop, grads, n, p, dtype, with_traffic)

    def alternative(self, grads, n, p, dtype, with_traffic=False):
        return self._sched(self.lib.ora_alternative, grads, n, p, dtype, with_traffic)

    def global_sync(self, grads, n, p, dtype):
        grads = np.ascontiguousarray(grads, NP[dtype])
        s, _, length = grads.shape
        chunk = (length + p - 1) // p
        out = np.zeros((n, chunk), NP[dtype])
        st = self.lib.ora_global_sync(_I(DTYPES[dtype]), _I(n), _I(p), _I(s), _SZ(length), _ptr(grads), _ptr(out))
        if st:
            raise OracleError(st)
        return out

    # ---- Adam
    class AdamScalars(C.Structure):
        _fields_ = [(k, C.c_float) for k in
                    ("b1", "omb1", "b2", "omb2", "eps", "wd", "step_size", "bc2_sqrt", "grad_scale")]

    def adam_scalars(self, lr, b1, b2, eps, wd, step, grad_scale):
        sc = Oracle.AdamScalars()
        self.lib.ora_adam_scalars(C.c_double(lr), C.c_double(b1), C.c_double(b2), C.c_double(eps), C.c_double(wd),
                                  _I(step), C.c_double(grad_scale), C.byref(sc))
        return sc

    def step1_shard(self, seed, n, p, s, j, segs, shard_elems, lr, b1=0.9, b2=0.999, eps=1e-8, wd=0.0,
                    threads=None):
        """Expected (master, m, v, bf16) of partition position j over its whole shard after
        one step of a generated-gradient step-driver job (ora_step1_shard, see the header).
        segs: (len, chunk, shard_off, grad_off) per layer."""
        sg = np.array([tuple(int(t) for t in x) for x in segs], np.uint64).reshape(-1, 4)
        out = [np.empty(shard_elems, np.float32) for _ in range(3)] + [np.empty(shard_elems, np.uint16)]
        th = threads or min(64, os.cpu_count() or 1)
        st = self.lib.ora_step1_shard(C.c_uint64(seed), _I(n), _I(p), _I(s), _I(j), _ptr(sg), _I(len(sg)),
                                      C.c_uint64(shard_elems), C.c_double(lr), C.c_double(b1), C.c_double(b2),
                                      C.c_double(eps), C.c_double(wd), _I(th), *[_ptr(a) for a in out])
        if st:
            raise OracleError(st, "step1_shard")
        return tuple(out)

    def adam(self, param, m, v, grad, lr, b1, b2, eps, wd, step, grad_scale=1.0, want_bf16=False):
        """Returns updated copies (param, m, v, param_bf16_or_None)."""
        param = np.array(param, np.float32)
        m = np.array(m, np.float32)
        v = np.array(v, np.float32)
        grad = np.ascontiguousarray(grad, np.float32)
        bf = np.empty(param.shape, np.uint16) if want_bf16 else None
        sc = self.adam_scalars(lr, b1, b2, eps, wd, step, grad_scale)
        self.lib.ora_adam_f32(_SZ(param.size), _ptr(param), _ptr(m), _ptr(v), _ptr(grad), C.byref(sc), _ptr(bf))
        return param, m, v, bf


class RefLib:
    """The unmodified reference (oracle/_ref).  ``RefLib.available()`` first."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    @staticmethod
    def _traffic(buf, nt):
        t = buf[: 3 * nt].reshape(-1, 3)
        return {(int(a), int(b)): int(c) for a, b, c in t}

    def random_shards(self, count, chunk, seed):
        out = np.empty(count * chunk, np.uint8)
        self.lib.ref_random_shards(_I(count), _SZ(chunk), C.c_uint32(seed), _ptr(out))
        return out.reshape(count, chunk)

    def random_i64(self, count, lo, hi, seed):
        out = np.empty(count, np.int64)
        self.lib.ref_random_i64(_SZ(count), C.c_int64(lo), C.c_int64(hi), C.c_uint32(seed), _ptr(out))
        return out

    def random_f32(self, count, lo, hi, seed):
        out = np.empty(count, np.float32)
        self.lib.ref_random_f32(_SZ(count), C.c_float(lo), C.c_float(hi), C.c_uint32(seed), _ptr(out))
        return out

    def build_group_layout(self, n, p):
        part = np.zeros(max(n, 1), np.int32)
        repl = np.zeros(max(n, 1), np.int32)
        self._check(self.lib.ref_build_group_layout(_I(n), _I(p), _ptr(part), _ptr(repl)))
        return part.reshape(n // p, p), repl.reshape(p, n // p)

    def partition_shape_ok(self, p, k):
        return bool(self.lib.ref_partition_shape_ok(_I(p), _I(k)))

    def min_feasible_partition(self, states, num_nodes, k, device_memory, node_granular, headroom=0.85):
        out = C.c_int(0)
        self._check(self.lib.ref_min_feasible_partition(C.c_uint64(states), _I(num_nodes), _I(k),
                                                        C.c_uint64(device_memory), _I(int(node_granular)),
                                                        C.c_double(headroom), C.byref(out)))
        return out.value

    def all_gather(self, shards, ranks=None, threads=1):
        shards = np.ascontiguousarray(shards, np.uint8)
        p, chunk = shards.shape
        ranks = np.arange(p, dtype=np.int32) if ranks is None else np.asarray(ranks, np.int32)
        out = np.empty((p, p * chunk), np.uint8)
        tb = np.zeros(3 * p * p + 3, np.int64)
        nt = C.c_int(0)
        self._check(self.lib.ref_all_gather(_I(threads), _ptr(ranks), _I(p), _ptr(shards), _SZ(chunk), _ptr(out),
                                            _ptr(tb), _I(p * p + 1), C.byref(nt)))
        return out, self._traffic(tb, nt.value)

    def reduce_scatter(self, bufs, dtype, ranks=None, threads=1):
        bufs = np.ascontiguousarray(bufs)
        p = bufs.shape[0]
        raw = bufs.view(np.uint8).reshape(p, -1)
        ranks = np.arange(p, dtype=np.int32) if ranks is None else np.asarray(ranks, np.int32)
        out = np.empty((p, raw.shape[1] // p), np.uint8)
        tb = np.zeros(3 * p * p + 3, np.int64)
        nt = C.c_int(0)
        self._check(self.lib.ref_reduce_scatter(_I(threads), _ptr(ranks), _I(p), _ptr(raw), _SZ(raw.shape[1]),
                                                _I(DTYPES[dtype]), _ptr(out), _ptr(tb), _I(p * p + 1), C.byref(nt)))
        return out.view(NP[dtype]), self._traffic(tb, nt.value)

    def all_reduce(self, bufs, dtype, ranks=None, threads=1):
        bufs = np.ascontiguousarray(bufs)
        p = bufs.shape[0]
        raw = bufs.view(np.uint8).reshape(p, -1)
        ranks = np.arange(p, dtype=np.int32) if ranks is None else np.asarray(ranks, np.int32)
        out = np.empty_like(raw)
        tb = np.zeros(3 * p * p + 3, np.int64)
        nt = C.c_int(0)
        self._check(self.lib.ref_all_reduce(_I(threads), _ptr(ranks), _I(p), _ptr(raw), _SZ(raw.shape[1]),
                                            _I(DTYPES[dtype]), _ptr(out), _ptr(tb), _I(p * p + 1), C.byref(nt)))
        return out.view(NP[dtype]), self._traffic(tb, nt.value)

    def hier_all_gather(self, shards, p, k, corrupt=False, threads=1):
        shards = np.ascontiguousarray(shards, np.uint8)
        n, chunk = shards.shape
        out = np.empty((n, p * chunk), np.uint8)
        tb = np.zeros(3 * n * n + 3, np.int64)
        nt = C.c_int(0)
        self._check(self.lib.ref_hier_all_gather(_I(threads), _I(n), _I(p), _I(k), _ptr(shards), _SZ(chunk),
                                                 _I(int(corrupt)), _ptr(out), _ptr(tb), _I(n * n + 1), C.byref(nt)))
        return out, self._traffic(tb, nt.value)

    def schedule(self, mode, grads, n, p, dtype, threads=1):
        """mode: 'two_hop' | 'alternative' | 'global_sync'.  Returns (shards, events, traffic)."""
        grads = np.ascontiguousarray(grads, NP[dtype])
        s, _, length = grads.shape
        chunk = (length + p - 1) // p
        out = np.zeros((n, chunk), NP[dtype])
        cap = s * n + n + 8
        ev = np.zeros(4 * cap, np.int64)
        nev = C.c_int(0)
        tb = np.zeros(3 * n * n + 3, np.int64)
        nt = C.c_int(0)
        fn = getattr(self.lib, f"ref_{mode}_{dtype}")
        self._check(fn(_I(threads), _I(n), _I(p), _I(s), _SZ(length), _ptr(grads), _ptr(out), _ptr(ev), _I(cap),
                       C.byref(nev), _ptr(tb), _I(n * n + 1), C.byref(nt)))
        return out, ev[: 4 * nev.value].reshape(-1, 4), self._traffic(tb, nt.value)

    def state_machine(self, n, p, s, length, ops: str):
        codes = np.zeros(len(ops), np.int32)
        self.lib.ref_state_machine(_I(n), _I(p), _I(s), _SZ(length), ops.encode(), _ptr(codes))
        return codes
