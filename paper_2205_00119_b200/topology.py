"""Scale-aware partitioning — the reference's topology layer
(topology.hpp:13-61, topology.cpp:7-84) over the C-ABI (host-only calls, no GPU).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from ._lib import Cluster, check, lib
from .workloads import transformer_layer_params  # noqa: F401  (re-exported)


@dataclass
class ClusterSpec:
    """topology.hpp:13-28 — node-major ranks: node_of(r) = r // k."""
    num_nodes: int = 1
    devices_per_node: int = 1
    intra_node_bandwidth: float = 0.0
    inter_node_bandwidth_per_node: float = 0.0
    alpha_intra: float = 0.0
    alpha_inter: float = 0.0
    device_memory: int = 0
    device_peak_flops: float = 0.0

    def total_ranks(self) -> int:
        return self.num_nodes * self.devices_per_node

    def node_of(self, rank: int) -> int:
        return rank // self.devices_per_node

    def local_node_rank(self, rank: int) -> int:
        return rank % self.devices_per_node

    def _c(self) -> Cluster:
        return Cluster(self.num_nodes, self.devices_per_node, self.intra_node_bandwidth,
                       self.inter_node_bandwidth_per_node, self.alpha_intra, self.alpha_inter,
                       self.device_memory, self.device_peak_flops)

    def validate(self) -> None:  # topology.cpp:7-19
        c = self._c()
        check(lib.mics_cluster_validate(C.byref(c)))


@dataclass
class GroupLayout:
    """topology.hpp:33-43: n/p contiguous partition groups, p stride-p replication groups."""
    n: int = 0
    p: int = 0
    partition_groups: list = field(default_factory=list)
    replication_groups: list = field(default_factory=list)

    def partition_group_of(self, rank: int) -> int:
        return rank // self.p

    def local_group_rank(self, rank: int) -> int:
        return rank % self.p

    def replication_group_of(self, rank: int) -> int:
        return rank % self.p

    def num_partition_groups(self) -> int:
        return self.n // self.p


def build_group_layout(n: int, p: int) -> GroupLayout:
    """topology.cpp:21-43 (OutOfRange / NonDivisible as the reference)."""
    size = max(n, 1)
    part = (C.c_int * size)()
    repl = (C.c_int * size)()
    check(lib.mics_build_group_layout(n, p, part, repl))
    return GroupLayout(
        n=n, p=p,
        partition_groups=[[part[g * p + i] for i in range(p)] for g in range(n // p)],
        replication_groups=[[repl[j * (n // p) + m] for m in range(n // p)] for j in range(p)])


def partition_shape_ok(p: int, k: int) -> bool:
    """topology.cpp:45-49."""
    return bool(lib.mics_partition_shape_ok(p, k))


def model_state_bytes(num_params: int, bytes_per_param_states: int = 16) -> int:
    """topology.cpp:51-56."""
    out = C.c_uint64(0)
    check(lib.mics_model_state_bytes(num_params, bytes_per_param_states, C.byref(out)))
    return out.value


def min_feasible_partition(model_state_bytes: int, cluster: ClusterSpec, node_granular: bool,
                           headroom_fraction: float = 0.85) -> int:
    """topology.cpp:58-84: smallest admissible p whose per-device share fits."""
    c = cluster._c()
    out = C.c_int(0)
    check(lib.mics_min_feasible_partition(model_state_bytes, C.byref(c), int(node_granular), headroom_fraction,
                                          C.byref(out)))
    return out.value
