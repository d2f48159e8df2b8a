"""Determinism across engine resources — the reference's contract that results and
the traffic log are bit-identical for any engine thread count
(collectives.hpp:38-41, test_collectives.cpp:179-207), restated for the GPU engine:
the "threads" are the CTAs per SM of every collective (Engine(num_threads) /
mics_set_parallelism), a forced small grid, the step's chained-gather CTAs per SM
(MICS_COPY_CTAS_PER_SM), graph replay vs eager enqueue, and barrier protocols.
Each variant is also compared with the CPU oracle (bit-exact), and the batched
collectives with the oracle directly (test_collectives.cpp:209-234)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (CTAs per SM, CTAs per launch): occupancy default, 1..4 per SM, and tiny grids
PARALLELISM = [(0, 0), (1, 0), (2, 0), (3, 0), (4, 0), (0, 7), (0, 1)]


@pytest.fixture(scope="module")
def m():
    import paper_2205_00119_b200 as m
    return m


def u8(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_collectives_identical_for_any_parallelism(m, oracle):
    """AG / RS (f32, p=8, many tiles) / AR / hierarchical AG (p=16, k=4) under every
    parallelism setting: identical bits and traffic, equal to the oracle."""
    eng = m.Engine(n_ranks=16, device=0, arena_bytes=1 << 30)
    rng = np.random.default_rng(5)
    ag_in = list(rng.integers(0, 256, (4, (3 << 20) + 7), dtype=np.uint8))
    rs_in = list(oracle.random_f32(8 * 8 * (1 << 19), -1.0, 1.0, 9).reshape(8, -1))
    ar_in = list(rng.standard_normal((4, 4 * 100_003)).astype(np.float64))
    hier_in = list(oracle.random_shards(16, 24 * 4099, 5))
    cluster = m.ClusterSpec(num_nodes=4, devices_per_node=4, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    want = {"ag": np.concatenate(ag_in), "rs": oracle.reduce_scatter(np.stack(rs_in), "f32"),
            "ar": oracle.all_reduce(np.stack(ar_in), "f64"),
            "hier": oracle.hier_all_gather(np.stack(hier_in), 16, 4)}
    first = None
    for cps, cap in PARALLELISM:
        eng.set_parallelism(cps, cap)
        eng.clear_traffic()
        got = {"ag": m.all_gather(eng, m.CollectiveGroup([0, 1, 2, 3]), ag_in),
               "rs": m.reduce_scatter(eng, m.CollectiveGroup(list(range(8, 16))), rs_in, "f32"),
               "ar": m.all_reduce(eng, m.CollectiveGroup([3, 7, 11, 15]), ar_in, "f64"),
               "hier": m.hierarchical_all_gather(eng, m.build_group_layout(16, 16), cluster, hier_in)}
        assert all(np.array_equal(o, want["ag"]) for o in got["ag"]), (cps, cap)
        assert np.array_equal(u8(np.stack(got["rs"])), u8(want["rs"])), (cps, cap)
        assert np.array_equal(u8(np.stack(got["ar"])), u8(want["ar"])), (cps, cap)
        assert np.array_equal(np.stack(got["hier"]), want["hier"]), (cps, cap)
        traffic = eng.traffic()
        if first is None:
            first = traffic
        assert traffic == first, (cps, cap)
    eng.close()


def test_reference_thread_case_on_every_grid(m, golden):
    """test_collectives.cpp:179-207 verbatim inputs (f32 RS p=8 on 16 floats from
    mt19937(9); hierarchical p=16, k=4, c=24, seed 5) with Engine(num_threads) = 1, 2,
    4, 8: the same bits as the reference's 1- and 8-thread golden outputs."""
    arr, dig = golden
    f = arr["kat/rs_f32_in"]
    cluster = m.ClusterSpec(num_nodes=4, devices_per_node=4, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    from oracle.oracle import Oracle
    shards = list(Oracle().random_shards(16, 24, 5))
    outs = []
    for threads in (1, 2, 4, 8):
        eng = m.Engine(threads, n_ranks=16, device=0, arena_bytes=16 << 20)
        out = m.reduce_scatter(eng, m.CollectiveGroup(list(range(8))), list(f), "f32")
        assert np.array_equal(u8(np.stack(out)), u8(arr["kat/rs_f32_out"]))
        assert np.array_equal(u8(np.stack(out)), u8(arr["kat/rs_f32_out_t8"]))
        outs.append((np.stack(m.hierarchical_all_gather(eng, m.build_group_layout(16, 16), cluster, shards)),
                     eng.traffic()))
        eng.close()
    for o, t in outs[1:]:
        assert np.array_equal(o, outs[0][0]) and t == outs[0][1]


def test_two_hop_sync_identical_for_any_parallelism(m, oracle):
    """The 2-hop schedule (s micro-step reduce-scatters + boundary all-reduce fused with
    Adam) under every parallelism setting: identical shards, parameters, Adam state
    and event log; equal to the oracle's two_hop."""
    from paper_2205_00119_b200.sync_schedule import AdamConfig, make_adam
    n, p, s, length = 8, 2, 3, 1_000_003
    g = oracle.random_f32(s * n * length, -1.0, 1.0, 17).reshape(s, n, length)
    red, _, _ = oracle.two_hop(g, n, p, "f32")
    res = []
    for cps, cap in PARALLELISM:
        eng = m.Engine(n_ranks=n, device=0, arena_bytes=512 << 20)
        eng.set_parallelism(cps, cap)
        lay = m.build_group_layout(n, p)
        st = m.make_sync_states(eng, lay, length, s, "f32")
        for t in range(s):
            m.two_hop_micro_step(eng, lay, st, list(g[t]))
        c = st.shard_elems
        bufs = [eng.alloc(4 * c) for _ in range(3)]
        for r in range(n):
            for b in bufs:
                eng.memset(b, r, 4 * c)
        log = []
        m.two_hop_boundary(eng, lay, st, log=log,
                           adam=make_adam(st, AdamConfig(lr=1e-3, grad_scale=1.0 / (n * s), write_grad=True), *bufs))
        eng.synchronize()
        got = [u8(eng.d2h(b, r, c)) for b in bufs for r in range(n)] + [u8(st.shard(r)) for r in range(n)]
        res.append((got, [(e.step, e.phase, e.group_id, e.bytes) for e in st.events()]))
        for r in range(n):
            assert np.array_equal(u8(st.shard(r)), u8(red[r])), (cps, cap, r)
        eng.close()
    for got, ev in res[1:]:
        assert ev == res[0][1]
        assert all(np.array_equal(a, b) for a, b in zip(got, res[0][0]))


@pytest.mark.parametrize("graph", ["1", "0"])
def test_step_identical_for_any_gather_grid(monkeypatch, graph):
    """The step driver with its chained per-layer gathers at 1-4 CTAs per SM, under a
    6-CTA launch cap, graph-replayed or eagerly enqueued: identical parameters,
    optimizer state and gather slots over two steps."""
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_GRAPH", graph)
    wl = Workload("det", [40_000, 9_001, 65_536, 4_099, 30_000, 12_288, 777], p=2, s=3)
    res = []
    for ctas, cap in ((1, 0), (2, 0), (3, 0), (4, 0), (0, 6)):
        monkeypatch.setenv("MICS_COPY_CTAS_PER_SM", str(ctas or 3))
        eng = Engine(n_ranks=8, device=0, arena_bytes=192 << 20)
        eng.set_parallelism(0, cap)
        step = MicsStep(eng, wl, StepOptions(seed=13))
        step.run(2)
        eng.synchronize()
        b, S = step.buffers(), step.sync_info()[0].shard_elems
        half, slots = step.stats().gather_slot_bytes, step.stats().gather_slots
        res.append([(u8(eng.d2h(b["master"], r, S)), u8(eng.d2h(b["exp_avg_sq"], r, S)),
                     u8(eng.d2h(b["gathered"], r, slots * half // 2, "bf16"))) for r in range(8)])
        step.close()
        eng.close()
    for other in res[1:]:
        for r in range(8):
            for a, c in zip(res[0][r], other[r]):
                assert np.array_equal(a, c), r


def test_batched_collectives_vs_oracle(m, oracle):
    """test_collectives.cpp:209-234 groups (0,2), (2,3), (5,1) plus a large group,
    batched in one launch, compared with the oracle's per-group results directly."""
    eng = m.Engine(n_ranks=8, device=0, arena_bytes=512 << 20)
    groups = [[0, 2], [2, 3], [5, 1], [4, 6, 7, 0]]
    for chunk in (1, 7, 4099, (1 << 20) + 5):
        sets = [oracle.random_shards(len(g), chunk, 3 + i) for i, g in enumerate(groups)]
        got = m.batched_all_gather(eng, [m.CollectiveGroup(g) for g in groups], [list(s) for s in sets])
        for g, s, out in zip(groups, sets, got):
            assert np.array_equal(np.stack(out), oracle.all_gather(s)), (g, chunk)
    for dtype in ("i64", "f32", "f64"):
        for chunk in (1, 5, 65_536 + 3):
            sets = []
            for i, g in enumerate(groups):
                if dtype == "i64":
                    sets.append(oracle.random_i64(len(g) * len(g) * chunk, -1000, 1000, 7 + i).reshape(len(g), -1))
                else:
                    x = oracle.random_f32(len(g) * len(g) * chunk, -1.0, 1.0, 7 + i).reshape(len(g), -1)
                    sets.append(x.astype(np.float64) if dtype == "f64" else x)
            got = m.batched_reduce_scatter(eng, [m.CollectiveGroup(g) for g in groups], [list(s) for s in sets], dtype)
            for g, s, out in zip(groups, sets, got):
                assert np.array_equal(u8(np.stack(out)), u8(oracle.reduce_scatter(s, dtype))), (dtype, g, chunk)
    eng.close()
