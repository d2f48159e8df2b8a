"""paper_2205_00119_b200 — B200-native MiCS communication hot path.

The package is a thin host layer over ``libmics.so`` (include/mics.h): hand-written
sm_100a kernels for the partition-group all-gather (flat and hierarchical), the
micro-step reduce-scatter, the boundary all-reduce fused with sharded Adam, over
NVLink peer memory.  The public names mirror the reference's sdpsim API.
"""
from .collectives import (CollectiveGroup, all_gather, all_reduce, batched_all_gather, batched_reduce_scatter,
                          hierarchical_all_gather, reduce_scatter)
from .engine import Engine
from .errors import Errc, Error
from .sync_schedule import (SyncEvent, SyncPhase, SyncStates, alternative_boundary, alternative_schedule_step,
                            make_sync_states, owned_chunk_elems, two_hop_boundary, two_hop_micro_step)
from .topology import (ClusterSpec, GroupLayout, build_group_layout, min_feasible_partition, model_state_bytes,
                       partition_shape_ok, transformer_layer_params)

VirtualRankEngine = Engine  # the reference's name for the transport

__all__ = [
    "Engine", "VirtualRankEngine", "Errc", "Error", "ClusterSpec", "GroupLayout", "build_group_layout",
    "partition_shape_ok", "model_state_bytes", "min_feasible_partition", "transformer_layer_params",
    "CollectiveGroup", "all_gather", "reduce_scatter", "all_reduce", "hierarchical_all_gather",
    "batched_all_gather", "batched_reduce_scatter", "SyncEvent", "SyncPhase", "SyncStates", "make_sync_states",
    "owned_chunk_elems", "two_hop_micro_step", "two_hop_boundary", "alternative_schedule_step",
    "alternative_boundary",
]
