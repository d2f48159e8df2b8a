"""Pin the CPU oracle (oracle/mics_oracle.c) to the reference's golden vectors.

The vectors were produced by the unmodified reference (tests/golden/make_golden.py);
these tests need no GPU and no /root/reference.  When oracle/_ref is present the
oracle is also cross-checked live against the reference on fresh inputs.
"""
import hashlib

import numpy as np
import pytest

from oracle.oracle import OracleError, RefLib


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


# ---------------------------------------------------------------- generators
def test_generators_match_libstdcxx(oracle, golden):
    arr, _ = golden
    for seed in (0, 1, 3, 5, 7, 11):
        assert np.array_equal(oracle.random_shards(4, 1024, seed).ravel(), arr[f"gen/shards/{seed}"])
    for seed in (1, 42, 2205, 1234):
        assert np.array_equal(oracle.random_i64(4096, -1000, 1000, seed), arr[f"gen/i64/{seed}"])
        assert np.array_equal(oracle.random_i64(512, -5, 5, seed), arr[f"gen/i64_5/{seed}"])
        assert np.array_equal(oracle.random_f32(4096, -1.0, 1.0, seed).view(np.uint32),
                              arr[f"gen/f32/{seed}"].view(np.uint32))


# ---------------------------------------------------------------- collectives KATs
def test_all_gather_kat(oracle, golden):
    arr, dig = golden
    out = oracle.all_gather(np.array([[1], [2], [3]], np.uint8))
    assert np.array_equal(out, arr["kat/ag_123"])
    assert (out == np.array([1, 2, 3], np.uint8)).all()
    t = oracle.traffic_all_gather([4, 5, 6, 7], 16, 8)
    expect = {(a, b): c for a, b, c in dig["kat/ag_traffic_4567"]}
    got = {(a, b): int(t[a, b]) for a in range(8) for b in range(8) if t[a, b]}
    assert got == expect
    for r in range(4, 8):
        assert int(t[:, r].sum()) == 3 * 16


def test_reduce_scatter_kats(oracle, golden):
    arr, dig = golden
    rs = oracle.reduce_scatter(np.array([[1, 2, 3, 4], [10, 20, 30, 40]], np.int64), "i64")
    assert np.array_equal(rs, arr["kat/rs_i64"])
    assert rs.tolist() == [[11, 22], [33, 44]]
    ar = oracle.all_reduce(np.array([[r, 10 * r, -r, 0] for r in range(4)], np.int64), "i64")
    assert np.array_equal(ar, arr["kat/ar_i64"])
    out = oracle.reduce_scatter(arr["kat/rs_f32_in"], "f32")
    assert np.array_equal(out.view(np.uint32), arr["kat/rs_f32_out"].view(np.uint32))
    assert np.array_equal(arr["kat/rs_f32_out"], arr["kat/rs_f32_out_t8"])
    with pytest.raises(OracleError) as e:
        oracle.reduce_scatter(np.zeros((2, 12), np.uint8), "i64")
    assert e.value.code == dig["err/ragged"] == 5  # TypeMismatch


# ---------------------------------------------------------------- hierarchical
def test_hierarchical_sweep_digests(oracle, golden):
    _, dig = golden
    for key, (d, total, inter) in dig["hier/sweep"].items():
        k, p, seed, chunk = map(int, key.split("/"))
        shards = oracle.random_shards(p, chunk, seed)
        out = oracle.hier_all_gather(shards, p, k)
        assert digest(out) == d, key
        assert np.array_equal(out, oracle.all_gather(shards))
        t = oracle.traffic_hier_all_gather(p, p, k, chunk)
        assert int(t.sum()) == total
        nodes = np.arange(p) // k
        assert int(t[nodes[:, None] != nodes[None, :]].sum()) == inter, key


def test_hierarchical_acceptance1_digests(oracle, golden):
    _, dig = golden
    for key, d in list(dig["acceptance1"].items())[::7]:  # every 7th case: keeps the CPU suite fast
        k, p, seed, chunk = map(int, key.split("/"))
        out = oracle.hier_all_gather(oracle.random_shards(p, chunk, seed * 977 + p), p, k)
        assert digest(out) == d, key


def test_hierarchical_layouts(oracle, golden):
    arr, dig = golden
    assert np.array_equal(oracle.hier_all_gather(arr["hier/multi_in"], 4, 2), arr["hier/multi_out"])
    c = oracle.hier_all_gather(np.arange(4, dtype=np.uint8).reshape(4, 1), 4, 2, corrupt=True)
    assert np.array_equal(c, arr["hier/corrupt_p4k2"])
    assert c[0].tolist() == [0, 2, 1, 3]  # PAPER.md:344-345 wrong layout
    c = oracle.hier_all_gather(np.arange(8, dtype=np.uint8).reshape(8, 1), 8, 4, corrupt=True)
    assert np.array_equal(c, arr["hier/corrupt_p8k4"])
    assert c[0].tolist() == [0, 4, 1, 5, 2, 6, 3, 7]
    c = oracle.hier_all_gather(oracle.random_shards(8, 3, 5), 4, 2, corrupt=True)
    assert np.array_equal(c, arr["hier/corrupt_n8p4k2_c3"])
    t = oracle.traffic_hier_all_gather(16, 16, 4, 32)
    expect = {(a, b): c for a, b, c in dig["hier/traffic_p16k4c32"]}
    assert {(a, b): int(t[a, b]) for a in range(16) for b in range(16) if t[a, b]} == expect
    nodes = np.arange(16) // 4
    assert int(t[nodes[:, None] != nodes[None, :]].sum()) == 16 * (16 - 4) // 4 * 32


# ---------------------------------------------------------------- sync schedule
def _i64(oracle, s, n, length, lo, hi, seed):
    return oracle.random_i64(s * n * length, lo, hi, seed).reshape(s, n, length)


def test_schedules_int64_sweep(oracle, golden):
    arr, _ = golden
    for n in (2, 4, 8, 16):
        for p in range(1, n + 1):
            if n % p:
                continue
            for s in (1, 2, 4):
                g = _i64(oracle, s, n, 13, -1000, 1000, n * 100 + p * 10 + s)
                th = oracle.two_hop(g, n, p, "i64")[0]
                alt = oracle.alternative(g, n, p, "i64")[0]
                gs = oracle.global_sync(g, n, p, "i64")
                assert np.array_equal(th, arr[f"sched/i64/{n}/{p}/{s}/two_hop"])
                assert np.array_equal(alt, arr[f"sched/i64/{n}/{p}/{s}/alternative"])
                assert np.array_equal(gs, arr[f"sched/i64/{n}/{p}/{s}/global_sync"])
                assert np.array_equal(th, gs)  # int64: exact equality (test_sync_schedule.cpp:54-57)


def test_schedules_acceptance2(oracle, golden):
    arr, _ = golden
    for n in (2, 4, 8, 16):
        for p in range(1, n + 1):
            if n % p:
                continue
            for s in (1, 2, 4):
                ga = _i64(oracle, s, n, 13, -1000, 1000, n * 1000 + p * 10 + s)
                assert np.array_equal(oracle.two_hop(ga, n, p, "i64")[0], arr[f"acc2/i64/{n}/{p}/{s}"])
                gf = oracle.random_f32(s * n * 13, -1.0, 1.0, n * 1000 + p * 10 + s).reshape(s, n, 13)
                for mode, fn in (("two_hop", oracle.two_hop), ("alternative", oracle.alternative)):
                    got = fn(gf, n, p, "f32")[0]
                    assert np.array_equal(got.view(np.uint32), arr[f"acc2/f32/{n}/{p}/{s}/{mode}"].view(np.uint32))
                gs = oracle.global_sync(gf, n, p, "f32")
                assert np.array_equal(gs.view(np.uint32), arr[f"acc2/f32/{n}/{p}/{s}/global_sync"].view(np.uint32))


def test_schedules_float_bitexact(oracle, golden):
    arr, _ = golden
    g = oracle.random_f32(3 * 8 * 21, -1.0, 1.0, 42).reshape(3, 8, 21)
    for mode, fn in (("two_hop", oracle.two_hop), ("alternative", oracle.alternative)):
        got = fn(g, 8, 4, "f32")[0]
        assert np.array_equal(got.view(np.uint32), arr[f"sched/f32/8/4/3/{mode}"].view(np.uint32))
        ref = arr["sched/f32/8/4/3/global_sync"]
        assert np.all(np.abs(got - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref)))  # :82-87
    g = oracle.random_f32(4 * 8 * 1001, -1.0, 1.0, 2205).reshape(4, 8, 1001)
    assert np.array_equal(oracle.two_hop(g, 8, 2, "f32")[0].view(np.uint32),
                          arr["sched/c1probe/two_hop"].view(np.uint32))
    assert np.array_equal(oracle.alternative(g, 8, 2, "f32")[0].view(np.uint32),
                          arr["sched/c1probe/alternative"].view(np.uint32))
    g64 = oracle.random_f32(2 * 4 * 10, -1.0, 1.0, 77).reshape(2, 4, 10).astype(np.float64)
    assert np.array_equal(oracle.two_hop(g64, 4, 2, "f64")[0], arr["sched/f64/two_hop"])


def test_schedule_events_and_traffic(oracle, golden):
    arr, dig = golden
    g = _i64(oracle, 2, 8, 16, -5, 5, 1)
    _, ev, tr = oracle.two_hop(g, 8, 4, "i64", with_traffic=True)
    assert np.array_equal(ev, arr["sched/events_two_hop"])
    micro = ev[ev[:, 1] == 0]
    assert len(micro) == 2 * 2 and (micro[:, 3] == 3 * 4 * 8).all()  # test_sync_schedule.cpp:104-114
    assert (ev[:, 1] == 1).sum() == 4
    expect = {(a, b): c for a, b, c in dig["sched/events_traffic"]}
    assert {(a, b): int(tr[a, b]) for a in range(8) for b in range(8) if tr[a, b]} == expect
    _, ev, _ = oracle.alternative(g, 8, 4, "i64")
    assert np.array_equal(ev, arr["sched/events_alt"])


# ---------------------------------------------------------------- topology
def test_topology(oracle, golden):
    arr, dig = golden
    for n in (4, 8, 12, 16, 24):
        for p in range(1, n + 1):
            if n % p == 0:
                part, repl = oracle.build_group_layout(n, p)
                assert np.array_equal(part, arr[f"topo/layout/{n}/{p}/part"])
                assert np.array_equal(repl, arr[f"topo/layout/{n}/{p}/repl"])
    for key, code in dig["topo/bad_layouts"].items():
        n, p = map(int, key.split("/"))
        with pytest.raises(OracleError) as e:
            oracle.build_group_layout(n, p)
        assert e.value.code == code
    for key, ok in dig["topo/shape_ok"].items():
        p, k = map(int, key.split("/"))
        assert oracle.partition_shape_ok(p, k) == ok
    for key, want in dig["topo/min_feasible"].items():
        states, nodes, k, mem, gran = map(int, key.split("/"))
        try:
            got = oracle.min_feasible_partition(states, nodes, k, mem, gran)
        except OracleError as e:
            got = -e.code
        assert got == want, key


# ---------------------------------------------------------------- live cross-check
@pytest.mark.skipif(not RefLib.available(), reason="oracle/_ref not built")
def test_live_against_reference(oracle):
    ref = RefLib()
    rng = np.random.default_rng(5)
    for n, p, k, chunk in ((8, 8, 4, 13), (8, 4, 2, 64), (16, 16, 4, 5), (12, 6, 3, 2)):
        shards = rng.integers(0, 256, (n, chunk), dtype=np.uint8)
        for corrupt in (False, True):
            assert np.array_equal(oracle.hier_all_gather(shards, p, k, corrupt),
                                  ref.hier_all_gather(shards, p, k, corrupt)[0])
    for n, p, s, length in ((8, 2, 4, 1001), (8, 8, 2, 77), (16, 4, 3, 130)):
        g = rng.standard_normal((s, n, length)).astype(np.float32)
        for mode, fn in (("two_hop", oracle.two_hop), ("alternative", oracle.alternative)):
            a, ev_a, tr_a = fn(g, n, p, "f32", with_traffic=True)
            b, ev_b, tr_b = ref.schedule(mode, g, n, p, "f32")
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
            assert np.array_equal(ev_a, ev_b)
            assert {(x, y): int(tr_a[x, y]) for x in range(n) for y in range(n) if tr_a[x, y]} == tr_b


def test_oracle_c1_full_size_matches_reference_digests(oracle, golden):
    """BASELINE config C1 at full size (4,198,400 params, n=8, p=2, s=4, mt19937(2205)
    U(-1,1)): the C restatement's two_hop and alternative shards hash to the digests
    the unmodified reference produced."""
    import hashlib
    arr, dig = golden
    n, p, s, length = 8, 2, 4, 4_198_400
    g = oracle.random_f32(s * n * length, -1.0, 1.0, 2205).reshape(s, n, length)
    for mode in ("two_hop", "alternative"):
        out = getattr(oracle, mode)(g, n, p, "f32")[0]
        assert [hashlib.sha256(np.ascontiguousarray(o).tobytes()).hexdigest()[:32] for o in out] == \
            dig[f"cfg/c1_full/{mode}"], mode
        assert np.array_equal(out[:, ::9973].view(np.uint32), arr[f"cfg/c1_full/{mode}_every_9973"].view(np.uint32))

