"""CPU-side checks of the drop-in boundary (no GPU calls):

* libmics.so loads and exports every entry point include/mics.h declares;
* the host-only topology entry points reproduce the reference's golden results
  (test_topology.cpp cases, via tests/golden);
* the Python mirror of the reference API raises the reference's errors.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mics.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:mics_status|int|const char\*)\s+(mics_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2205_00119_b200._lib import EXPORTS, LIB_PATH
    lib = C.CDLL(LIB_PATH)
    syms = declared_symbols()
    assert len(syms) > 60
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(EXPORTS), set(syms) ^ set(EXPORTS)
    assert lib.mics_abi_version() == 3


def test_status_names_follow_errc_order():
    from paper_2205_00119_b200._lib import lib
    from paper_2205_00119_b200.errors import Errc
    for e in Errc:
        assert lib.mics_status_name(int(e)).decode() == e.name


def test_topology_layouts_match_reference(golden):
    import paper_2205_00119_b200 as m
    arr, dig = golden
    for n in (4, 8, 12, 16, 24):
        for p in range(1, n + 1):
            if n % p == 0:
                lay = m.build_group_layout(n, p)
                assert np.array_equal(np.array(lay.partition_groups), arr[f"topo/layout/{n}/{p}/part"])
                assert np.array_equal(np.array(lay.replication_groups), arr[f"topo/layout/{n}/{p}/repl"])
                for r in range(n):
                    assert lay.partition_group_of(r) == r // p and lay.replication_group_of(r) == r % p
    for key, code in dig["topo/bad_layouts"].items():
        n, p = map(int, key.split("/"))
        with pytest.raises(m.Error) as e:
            m.build_group_layout(n, p)
        assert int(e.value.code) == code
        assert str(e.value).startswith(e.value.code.name + ": ")


def test_topology_shape_and_feasibility(golden):
    import paper_2205_00119_b200 as m
    _, dig = golden
    for key, ok in dig["topo/shape_ok"].items():
        p, k = map(int, key.split("/"))
        assert m.partition_shape_ok(p, k) == ok
    for key, want in dig["topo/min_feasible"].items():
        states, nodes, k, mem, gran = map(int, key.split("/"))
        c = m.ClusterSpec(num_nodes=nodes, devices_per_node=k, intra_node_bandwidth=1,
                          inter_node_bandwidth_per_node=1, device_memory=mem)
        try:
            got = m.min_feasible_partition(states, c, bool(gran))
        except m.Error as e:
            got = -int(e.code)
        assert got == want, key
    assert m.model_state_bytes(1_000_000) == 16_000_000
    assert m.model_state_bytes(10, 4) == 40
    with pytest.raises(m.Error):
        m.model_state_bytes(0)


def test_cluster_validation():
    import paper_2205_00119_b200 as m
    c = m.ClusterSpec(num_nodes=2, devices_per_node=4, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    c.validate()
    assert c.total_ranks() == 8 and c.node_of(5) == 1 and c.local_node_rank(5) == 1
    c.num_nodes = 0
    with pytest.raises(m.Error) as e:
        c.validate()
    assert e.value.code == m.Errc.OutOfRange


def test_group_validation_and_transformer_shapes():
    import paper_2205_00119_b200 as m
    with pytest.raises(m.Error) as e:
        m.CollectiveGroup([0, 1, 1]).validate()
    assert e.value.code == m.Errc.ShapeError
    # SURVEY §8 config shapes from the reference's derive_layers_from_transformer
    assert sum(m.transformer_layer_params(1024, 4096, 24, 30522, 512)) == 334_088_192
    assert sum(m.transformer_layer_params(1600, 6400, 48, 50257, 1024)) == 1_557_608_000
    assert sum(m.transformer_layer_params(2560, 10240, 127, 32008, 512)) == 10_075_164_160


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2205_00119_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                for bad in ("from oracle", "import oracle", "liboracle", "libsdpsim_ref"):
                    assert bad not in text, (f, bad)
