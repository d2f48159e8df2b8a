"""ctypes binding of libmics.so (include/mics.h).

The product path has no fallback: if the CUDA library is missing this module
raises at import time, and every call that fails on the device raises
:class:`paper_2205_00119_b200.errors.Error` with the library's message.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmics.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or `make -C paper_2205_00119_b200/csrc`)")

lib = C.CDLL(LIB_PATH)

VP = C.c_void_p
I = C.c_int
U64 = C.c_uint64
I64 = C.c_int64
D = C.c_double
PI = C.POINTER(C.c_int)
PU64 = C.POINTER(C.c_uint64)
PVP = C.POINTER(C.c_void_p)

IPC_HANDLE_BYTES = 64
MAX_WORLD = 64


class Buf(C.Structure):
    """mics_buf: a symmetric allocation (offset, stride)."""
    _fields_ = [("offset", U64), ("stride", U64)]


class Cluster(C.Structure):
    _fields_ = [("num_nodes", I), ("devices_per_node", I), ("intra_node_bandwidth", D),
                ("inter_node_bandwidth_per_node", D), ("alpha_intra", D), ("alpha_inter", D),
                ("device_memory", U64), ("device_peak_flops", D)]


class InitArgs(C.Structure):
    _fields_ = [("n_ranks", I), ("world", I), ("world_rank", I), ("device", I), ("arena_bytes", U64)]


class AgDesc(C.Structure):
    _fields_ = [("ranks", PI), ("p", I), ("d_shard", PVP), ("chunk_bytes", U64), ("d_out", PVP)]


class RsDesc(C.Structure):
    _fields_ = [("ranks", PI), ("p", I), ("d_in", PVP), ("in_elems", U64), ("valid_elems", U64), ("d_out", PVP)]


class SyncInfo(C.Structure):
    _fields_ = [("n", I), ("p", I), ("s", I), ("nseg", I), ("micro_step", I), ("acc_t", I),
                ("shard_elems", U64), ("grad_elems", U64), ("boundary_sub", U64), ("shard", Buf)]


class Adam(C.Structure):
    _fields_ = [("lr", D), ("beta1", D), ("beta2", D), ("eps", D), ("weight_decay", D), ("step", I),
                ("grad_scale", D), ("param", Buf), ("exp_avg", Buf), ("exp_avg_sq", Buf), ("param_bf16", Buf),
                ("write_grad", I)]


class StepCfg(C.Structure):
    _fields_ = [("p", I), ("s", I), ("nlayers", I), ("layer_params", PU64), ("grad_t", I), ("hier_k", I),
                ("resident_grads", I), ("alternative", I), ("seed", U64), ("lr", D), ("beta1", D), ("beta2", D),
                ("eps", D), ("weight_decay", D), ("compute", I), ("recompute", I), ("tokens", U64), ("hidden", U64)]


class StepStats(C.Structure):
    _fields_ = [("ag_bytes_in", U64), ("rs_bytes_in", U64), ("ar_bytes_in", U64), ("adam_hbm_bytes", U64),
                ("gen_bytes", U64), ("launches", U64), ("shard_elems", U64), ("gathered_max_bytes", U64),
                ("grad_elems", U64), ("adam_step", I),
                ("ag_remote_bytes", U64), ("ag_hbm_bytes", U64), ("ag_launches", U64),
                ("rs_remote_bytes", U64), ("rs_hbm_bytes", U64), ("rs_launches", U64),
                ("bnd_remote_bytes", U64), ("bnd_hbm_bytes", U64), ("bnd_launches", U64),
                ("compute_flops", D), ("gemm_launches", U64), ("gather_slots", U64), ("gather_slot_bytes", U64)]


# (name, restype, argtypes); restype I is a mics_status
_SIGS = [
    ("mics_status_name", C.c_char_p, [I]),
    ("mics_last_error", C.c_char_p, []),
    ("mics_abi_version", I, []),
    ("mics_build_group_layout", I, [I, I, PI, PI]),
    ("mics_partition_shape_ok", I, [I, I]),
    ("mics_model_state_bytes", I, [U64, U64, PU64]),
    ("mics_cluster_validate", I, [C.POINTER(Cluster)]),
    ("mics_min_feasible_partition", I, [U64, C.POINTER(Cluster), I, D, PI]),
    ("mics_init", I, [C.POINTER(InitArgs), C.POINTER(VP)]),
    ("mics_init_devices", I, [C.POINTER(InitArgs), PI, I, C.POINTER(VP)]),
    ("mics_device_count", I, [VP, PI]),
    ("mics_device_stream", I, [VP, I, C.POINTER(VP)]),
    ("mics_destroy", I, [VP]),
    ("mics_ipc_export", I, [VP, VP]),
    ("mics_ipc_import", I, [VP, VP]),
    ("mics_rank_process", I, [VP, I, PI]),
    ("mics_local_ranks", I, [VP, PI, PI]),
    ("mics_set_parallelism", I, [VP, I, I]),
    ("mics_alloc", I, [VP, U64, C.POINTER(Buf)]),
    ("mics_arena_mark", I, [VP, PU64]),
    ("mics_arena_release", I, [VP, U64]),
    ("mics_arena_used", I, [VP, PU64, PU64]),
    ("mics_buf_ptr", I, [VP, Buf, I, C.POINTER(VP)]),
    ("mics_memset", I, [VP, Buf, I, U64, I, U64]),
    ("mics_h2d", I, [VP, Buf, I, U64, VP, U64]),
    ("mics_d2h", I, [VP, Buf, I, U64, VP, U64]),
    ("mics_stream", I, [VP, C.POINTER(VP)]),
    ("mics_synchronize", I, [VP]),
    ("mics_barrier", I, [VP]),
    ("mics_launch_count", I, [VP, PU64]),
    ("mics_num_sms", I, [VP, PI]),
    ("mics_host_alloc", I, [U64, C.POINTER(VP)]),
    ("mics_host_free", I, [VP]),
    ("mics_traffic_enable", I, [VP, I]),
    ("mics_traffic_clear", I, [VP]),
    ("mics_traffic_size", I, [VP, PU64]),
    ("mics_traffic_get", I, [VP, C.POINTER(I64), U64]),
    ("mics_all_gather", I, [VP, PI, I, PVP, U64, PVP]),
    ("mics_reduce_scatter", I, [VP, PI, I, PVP, U64, U64, I, I, D, I, PVP]),
    ("mics_all_reduce", I, [VP, PI, I, PVP, U64, I]),
    ("mics_hier_all_gather", I, [VP, I, I, PVP, U64, PVP, I]),
    ("mics_batched_all_gather", I, [VP, C.POINTER(AgDesc), I]),
    ("mics_batched_reduce_scatter", I, [VP, C.POINTER(RsDesc), I, I, I, D, I]),
    ("mics_plan_all_gather", I, [VP, PI, I, PVP, U64, PVP, C.POINTER(VP)]),
    ("mics_plan_reduce_scatter", I, [VP, PI, I, PVP, U64, U64, I, I, D, I, PVP, C.POINTER(VP)]),
    ("mics_plan_run", I, [VP, VP, I]),
    ("mics_plan_destroy", I, [VP]),
    ("mics_host_all_gather", I, [VP, PI, I, PVP, U64, PVP]),
    ("mics_host_reduce_scatter", I, [VP, PI, I, PVP, U64, I, PVP]),
    ("mics_host_all_reduce", I, [VP, PI, I, PVP, U64, I, PVP]),
    ("mics_host_hier_all_gather", I, [VP, I, I, I, PVP, U64, PVP, I]),
    ("mics_host_batched_all_gather", I, [VP, I, PI, PI, PU64, PVP, PVP]),
    ("mics_host_batched_reduce_scatter", I, [VP, I, PI, PI, PU64, PVP, I, PVP]),
    ("mics_sync_create", I, [VP, I, I, I, PU64, I, C.c_uint32, C.POINTER(VP)]),
    ("mics_sync_destroy", I, [VP]),
    ("mics_sync_get_info", I, [VP, C.POINTER(SyncInfo)]),
    ("mics_sync_seg", I, [VP, I, PU64, PU64, PU64, PU64]),
    ("mics_sync_micro_step", I, [VP, VP, Buf, U64, I, D, I]),
    ("mics_sync_boundary", I, [VP, VP, C.POINTER(Adam)]),
    ("mics_sync_alt_step", I, [VP, VP, Buf, U64, I, D]),
    ("mics_sync_alt_boundary", I, [VP, VP]),
    ("mics_sync_events", I, [VP, C.POINTER(I64), U64, PU64]),
    ("mics_sync_clear_events", I, [VP]),
    ("mics_generate", I, [VP, Buf, I, U64, I, U64, I, I, U64, U64]),
    ("mics_step_create", I, [VP, C.POINTER(StepCfg), C.POINTER(VP)]),
    ("mics_step_destroy", I, [VP]),
    ("mics_step_run", I, [VP, VP, I]),
    ("mics_step_stats_get", I, [VP, C.POINTER(StepStats)]),
    ("mics_step_sync", I, [VP, C.POINTER(VP)]),
    ("mics_step_buffers", I, [VP] + [C.POINTER(Buf)] * 6),
    ("mics_step_profile", I, [VP, VP] + [C.POINTER(D)] * 4),
    ("mics_step_run_host", I, [VP, VP, VP, I, VP]),
    ("mics_step_profile_ex", I, [VP, VP, C.POINTER(D)]),
    ("mics_gemm_bf16", I, [VP, VP, U64, I, VP, U64, I, VP, U64, I, I, I, I, I]),
]

EXPORTS = [name for name, _, _ in _SIGS]

for _name, _res, _args in _SIGS:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def check(status: int) -> None:
    """Raise the library's error for a non-zero mics_status."""
    if status:
        from .errors import Error
        raise Error(int(status), lib.mics_last_error().decode())
