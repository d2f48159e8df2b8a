"""paper_2205_00119_b200 — B200-native MiCS communication hot path.

The package is a thin host layer over ``libmics.so`` (include/mics.h): hand-written
sm_100a kernels for the partition-group all-gather (flat and hierarchical), the
micro-step reduce-scatter, the boundary all-reduce fused with sharded Adam, over
NVLink peer memory.  The public names mirror the reference's sdpsim API.

Names are resolved lazily (PEP 562): ``import paper_2205_00119_b200.workloads``
describes the BASELINE jobs without loading the native library, while touching
any API name imports its module, and with it ``_lib``, which raises when
``libmics.so`` is missing — there is no CPU fallback.
"""
from __future__ import annotations

import importlib

_EXPORTS = {
    "collectives": ("CollectiveGroup", "all_gather", "all_reduce", "batched_all_gather", "batched_reduce_scatter",
                    "hierarchical_all_gather", "reduce_scatter"),
    "engine": ("Engine",),
    "errors": ("Errc", "Error"),
    "sync_schedule": ("SyncEvent", "SyncPhase", "SyncStates", "alternative_boundary", "alternative_schedule_step",
                      "make_sync_states", "owned_chunk_elems", "two_hop_boundary", "two_hop_micro_step"),
    "topology": ("ClusterSpec", "GroupLayout", "build_group_layout", "min_feasible_partition", "model_state_bytes",
                 "partition_shape_ok"),
    "workloads": ("transformer_layer_params", "Workload", "workloads"),
}
_WHERE = {name: mod for mod, names in _EXPORTS.items() for name in names}
_WHERE["VirtualRankEngine"] = "engine"  # the reference's name for the transport

__all__ = sorted(_WHERE)


def __getattr__(name: str):
    mod = _WHERE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(importlib.import_module(f".{mod}", __name__), "Engine" if name == "VirtualRankEngine" else name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(_WHERE))
