"""GPU parity: libmics (sm_100a kernels through the C-ABI) against the CPU oracle
and the reference's golden vectors — the reference's own unit tests
(test_collectives.cpp, test_sync_schedule.cpp) restated over the B200 engine.

Bit-exact for bytes and integers; bit-exact for floats too, because the pull
kernels fold in the reference's ascending-position order.
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.fixture(scope="module")
def m():
    import paper_2205_00119_b200 as m
    return m


@pytest.fixture(scope="module", params=["1gpu", "2gpus_one_process"])
def engines(m, request):
    """Engines of n virtual ranks on GPU 0, or spread node-major over GPUs 0 and 1 of
    this one process (mics_init_devices): every test below runs on both."""
    devices = None
    if request.param == "2gpus_one_process":
        import torch
        if torch.cuda.device_count() < 2:
            pytest.skip("needs 2 GPUs")
        devices = [0, 1]
    cache = {}

    def get(n):
        if n not in cache:
            cache[n] = m.Engine(n_ranks=n, device=0, arena_bytes=512 << 20, devices=devices)
        cache[n].clear_traffic()
        return cache[n]
    yield get
    for e in cache.values():
        e.close()


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


# ------------------------------------------------------------------ collectives (test_collectives.cpp)
def test_all_gather_concatenates_in_group_order(m, engines, golden):
    arr, _ = golden
    eng = engines(64)
    out = m.all_gather(eng, m.CollectiveGroup([0, 1, 2]), [b"\x01", b"\x02", b"\x03"])
    for o in out:
        assert o.tolist() == [1, 2, 3]
    assert np.array_equal(np.stack(out), arr["kat/ag_123"])


def test_all_gather_traffic_log(m, engines, oracle, golden):
    _, dig = golden
    eng = engines(64)
    m.all_gather(eng, m.CollectiveGroup([4, 5, 6, 7]), list(oracle.random_shards(4, 16, 7)))
    t = eng.traffic()
    assert t == {(a, b): c for a, b, c in dig["kat/ag_traffic_4567"]}
    for r in (4, 5, 6, 7):
        assert eng.bytes_received_by(r) == 3 * 16
    assert all(a != b for a, b in t) and sum(t.values()) == 4 * 3 * 16


def test_reduce_scatter_kat_and_errors(m, engines):
    eng = engines(64)
    g = m.CollectiveGroup([0, 1])
    out = m.reduce_scatter(eng, g, [np.array([1, 2, 3, 4], np.int64), np.array([10, 20, 30, 40], np.int64)], "i64")
    assert out[0].tolist() == [11, 22] and out[1].tolist() == [33, 44]
    m.reduce_scatter(eng, g, [np.zeros(32, np.uint8), np.zeros(32, np.uint8)], "i64")
    with pytest.raises(m.Error) as e:
        m.reduce_scatter(eng, g, [np.zeros(16, np.uint8), np.zeros(24, np.uint8)], "i64")
    assert e.value.code == m.Errc.SizeMismatch
    with pytest.raises(m.Error) as e:
        m.reduce_scatter(eng, g, [np.zeros(12, np.uint8), np.zeros(12, np.uint8)], "i64")
    assert e.value.code == m.Errc.TypeMismatch
    with pytest.raises(m.Error) as e:
        m.all_gather(eng, m.CollectiveGroup([0, 1, 1]), [b"a", b"b", b"c"])
    assert e.value.code == m.Errc.ShapeError


def test_all_reduce_full_sum(m, engines, golden):
    arr, _ = golden
    eng = engines(64)
    bufs = [np.array([r, 10 * r, -r, 0], np.int64) for r in range(4)]
    out = m.all_reduce(eng, m.CollectiveGroup([0, 1, 2, 3]), bufs, "i64")
    for o in out:
        assert o.tolist() == [6, 60, -6, 0]
    assert np.array_equal(np.stack(out), arr["kat/ar_i64"])


def test_reduce_scatter_float_is_bitexact_and_thread_independent(m, engines, golden):
    arr, _ = golden
    f = arr["kat/rs_f32_in"]
    for threads in (1, 8):
        eng = m.Engine(threads, n_ranks=8, device=0, arena_bytes=16 << 20)
        out = m.reduce_scatter(eng, m.CollectiveGroup(list(range(8))), list(f), "f32")
        assert np.array_equal(u32(np.stack(out)), u32(arr["kat/rs_f32_out"]))
        eng.close()


@pytest.mark.parametrize("dtype", ["i64", "f32", "f64"])
@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_reduce_scatter_random_vs_oracle(m, engines, oracle, dtype, p):
    eng = engines(64)
    rng = np.random.default_rng(p)
    for chunk in (1, 5, 1024, 4099, 65536 + 3):
        if dtype == "i64":
            bufs = rng.integers(-(1 << 40), 1 << 40, (p, p * chunk), dtype=np.int64)
        else:
            bufs = rng.standard_normal((p, p * chunk)).astype({"f32": np.float32, "f64": np.float64}[dtype])
        ranks = list(range(10, 10 + p))
        out = m.reduce_scatter(eng, m.CollectiveGroup(ranks), list(bufs), dtype)
        want = oracle.reduce_scatter(bufs, dtype)
        assert np.array_equal(np.stack(out).view(np.uint8), want.view(np.uint8)), (dtype, p, chunk)


def test_hierarchical_matches_flat_sweep(m, engines, oracle, golden):
    """test_collectives.cpp:98-121 — k in {1,2,4,8}, p = k..64 step k, seeds {0,1}, chunk {1,7}."""
    _, dig = golden
    eng = engines(64)
    for key, (d, total, inter) in dig["hier/sweep"].items():
        k, p, seed, chunk = map(int, key.split("/"))
        cl = m.ClusterSpec(num_nodes=p // k, devices_per_node=k, intra_node_bandwidth=1,
                           inter_node_bandwidth_per_node=1)
        lay = m.build_group_layout(p, p)
        shards = oracle.random_shards(p, chunk, seed)
        eng.clear_traffic()
        out = m.hierarchical_all_gather(eng, lay, cl, list(shards))
        assert digest(np.stack(out)) == d, key
        t = eng.traffic()
        assert sum(t.values()) == total
        assert sum(c for (a, b), c in t.items() if a // k != b // k) == inter, key


def test_hierarchical_acceptance1(m, engines, oracle, golden):
    """acceptance_main.cpp:50-88 (1800 cases incl. chunk 1024) — and under the reference's 30 s limit."""
    import time
    _, dig = golden
    eng = engines(64)
    eng.enable_traffic(False)
    t0 = time.time()
    for key, d in dig["acceptance1"].items():
        k, p, seed, chunk = map(int, key.split("/"))
        cl = m.ClusterSpec(num_nodes=p // k, devices_per_node=k, intra_node_bandwidth=1,
                           inter_node_bandwidth_per_node=1)
        out = m.hierarchical_all_gather(eng, m.build_group_layout(p, p), cl,
                                        list(oracle.random_shards(p, chunk, seed * 977 + p)))
        assert digest(np.stack(out)) == d, key
    eng.enable_traffic(True)
    assert time.time() - t0 < 30.0


def test_hierarchical_multigroup_and_corrupt(m, engines, oracle, golden):
    arr, dig = golden
    eng = engines(8)
    cl = m.ClusterSpec(num_nodes=4, devices_per_node=2, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    out = m.hierarchical_all_gather(eng, m.build_group_layout(8, 4), cl, list(arr["hier/multi_in"]))
    assert np.array_equal(np.stack(out), arr["hier/multi_out"])
    # corrupt-stage2 hook: [C0, C2, C1, C3] (test_collectives.cpp:142-158)
    cl4 = m.ClusterSpec(num_nodes=2, devices_per_node=2, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    out = m.hierarchical_all_gather(eng, m.build_group_layout(4, 4), cl4, [b"\x00", b"\x01", b"\x02", b"\x03"],
                                    corrupt_stage2=True)
    for o in out:
        assert o.tolist() == [0, 2, 1, 3]
    cl8 = m.ClusterSpec(num_nodes=2, devices_per_node=4, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    out = m.hierarchical_all_gather(eng, m.build_group_layout(8, 8), cl8, [bytes([i]) for i in range(8)],
                                    corrupt_stage2=True)
    assert np.array_equal(np.stack(out), arr["hier/corrupt_p8k4"])
    out = m.hierarchical_all_gather(eng, m.build_group_layout(8, 4), cl, list(oracle.random_shards(8, 3, 5)),
                                    corrupt_stage2=True)
    assert np.array_equal(np.stack(out), arr["hier/corrupt_n8p4k2_c3"])
    # inter-node traffic p=16, k=4 (test_collectives.cpp:160-177)
    e16 = engines(16)
    cl16 = m.ClusterSpec(num_nodes=4, devices_per_node=4, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    m.hierarchical_all_gather(e16, m.build_group_layout(16, 16), cl16, list(oracle.random_shards(16, 32, 11)))
    assert e16.traffic() == {(a, b): c for a, b, c in dig["hier/traffic_p16k4c32"]}
    cl6 = m.ClusterSpec(num_nodes=1, devices_per_node=6, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    with pytest.raises(m.Error) as e:
        m.hierarchical_all_gather(eng, m.build_group_layout(6, 6), cl6, [b"x"] * 5)
    assert e.value.code == m.Errc.SizeMismatch
    cl3 = m.ClusterSpec(num_nodes=4, devices_per_node=3, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    with pytest.raises(m.Error) as e:  # p=4 is not node-aligned for k=3 (collectives.cpp:208-210)
        m.hierarchical_all_gather(engines(64), m.build_group_layout(12, 4), cl3, [b"x"] * 12)
    assert e.value.code == m.Errc.ShapeError


@pytest.mark.parametrize("corrupt", [False, True])
def test_hierarchical_multi_tile_vs_oracle(m, oracle, corrupt):
    """k_hier with chunks of many 32 KiB tiles (stage-3 tiles wait on per-tile flags of
    the node peers' stage-1 tiles), aligned and byte-ragged, several partition groups,
    the wrong-layout hook included, under full and tiny grids."""
    eng = m.Engine(n_ranks=16, device=0, arena_bytes=1 << 30)
    for n, p, k, chunk in ((16, 8, 4, (1 << 20) + 3), (16, 8, 2, 4 << 20), (16, 16, 4, 300_000), (8, 4, 2, 65_536)):
        shards = oracle.random_shards(n, chunk, n + p + k)
        want = oracle.hier_all_gather(shards, p, k, corrupt)
        cl = m.ClusterSpec(num_nodes=n // k, devices_per_node=k, intra_node_bandwidth=1,
                           inter_node_bandwidth_per_node=1)
        for cps, cap in ((0, 0), (1, 0), (0, 3)):
            eng.set_parallelism(cps, cap)
            got = m.hierarchical_all_gather(eng, m.build_group_layout(n, p), cl, list(shards), corrupt_stage2=corrupt)
            assert np.array_equal(np.stack(got), want), (n, p, k, chunk, cps, cap)
    eng.close()


def test_batched_equals_sequential(m, engines, oracle):
    eng = engines(64)
    groups = [m.CollectiveGroup([0, 1]), m.CollectiveGroup([2, 3, 4]), m.CollectiveGroup([5])]
    sets = [list(oracle.random_shards(g.size(), 8, s)) for s, g in enumerate(groups)]
    batched = m.batched_all_gather(eng, groups, sets)
    for g, s, b in zip(groups, sets, batched):
        seq = m.all_gather(eng, g, s)
        assert all(np.array_equal(x, y) for x, y in zip(b, seq))
    bsets = [[np.full(g.size() * 2, r + 1, np.int64) for r in range(g.size())] for g in groups]
    brs = m.batched_reduce_scatter(eng, groups, bsets, "i64")
    for g, s, b in zip(groups, bsets, brs):
        seq = m.reduce_scatter(eng, g, s, "i64")
        assert all(np.array_equal(x, y) for x, y in zip(b, seq))
    assert m.batched_all_gather(eng, [], []) == []


def test_large_unaligned_and_aligned_all_gather(m, engines):
    eng = engines(8)
    rng = np.random.default_rng(0)
    for p, chunk in ((2, (32 << 20) + 3), (8, 4 << 20), (4, 1 << 20)):
        shards = rng.integers(0, 256, (p, chunk), dtype=np.uint8)
        out = m.all_gather(eng, m.CollectiveGroup(list(range(p))), list(shards))
        flat = shards.reshape(-1)
        for o in out:
            assert np.array_equal(o, flat)


# ------------------------------------------------------------------ sync schedule (test_sync_schedule.cpp)
def test_schedules_int64_sweep(m, engines, oracle, golden):
    arr, _ = golden
    for n in (2, 4, 8, 16):
        eng = engines(n)
        for p in range(1, n + 1):
            if n % p:
                continue
            lay = m.build_group_layout(n, p)
            for s in (1, 2, 4):
                g = oracle.random_i64(s * n * 13, -1000, 1000, n * 100 + p * 10 + s).reshape(s, n, 13)
                th = m.make_sync_states(eng, lay, 13, s, "i64")
                for t in range(s):
                    m.two_hop_micro_step(eng, lay, th, list(g[t]))
                m.two_hop_boundary(eng, lay, th)
                alt = m.make_sync_states(eng, lay, 13, s, "i64")
                for t in range(s):
                    m.alternative_schedule_step(eng, lay, alt, list(g[t]))
                m.alternative_boundary(alt)
                want = arr[f"sched/i64/{n}/{p}/{s}/global_sync"]
                for r in range(n):
                    assert np.array_equal(th.shard(r), want[r]), (n, p, s, r)
                    assert np.array_equal(alt.shard(r), want[r]), (n, p, s, r)
                th.close()
                alt.close()


def test_schedules_float_bitexact_with_reference(m, engines, oracle, golden):
    arr, _ = golden
    eng = engines(8)
    lay = m.build_group_layout(8, 4)
    g = oracle.random_f32(3 * 8 * 21, -1.0, 1.0, 42).reshape(3, 8, 21)
    th = m.make_sync_states(eng, lay, 21, 3, "f32")
    alt = m.make_sync_states(eng, lay, 21, 3, "f32")
    for t in range(3):
        m.two_hop_micro_step(eng, lay, th, list(g[t]))
        m.alternative_schedule_step(eng, lay, alt, list(g[t]))
    m.two_hop_boundary(eng, lay, th)
    m.alternative_boundary(alt)
    ref = arr["sched/f32/8/4/3/global_sync"]
    for r in range(8):
        assert np.array_equal(u32(th.shard(r)), u32(arr["sched/f32/8/4/3/two_hop"][r]))
        assert np.array_equal(u32(alt.shard(r)), u32(arr["sched/f32/8/4/3/alternative"][r]))
        assert np.all(np.abs(th.shard(r) - ref[r]) <= 1e-5 * np.maximum(1.0, np.abs(ref[r])))
    # C1-shaped probe n=8, p=2, s=4, len 1001 (bit-exact with pinned order)
    lay = m.build_group_layout(8, 2)
    g = oracle.random_f32(4 * 8 * 1001, -1.0, 1.0, 2205).reshape(4, 8, 1001)
    th = m.make_sync_states(eng, lay, 1001, 4, "f32")
    for t in range(4):
        m.two_hop_micro_step(eng, lay, th, list(g[t]))
    m.two_hop_boundary(eng, lay, th)
    for r in range(8):
        assert np.array_equal(u32(th.shard(r)), u32(arr["sched/c1probe/two_hop"][r]))


def test_schedule_acceptance2_float(m, engines, oracle, golden):
    arr, _ = golden
    for n in (2, 4, 8, 16):
        eng = engines(n)
        for p in [q for q in range(1, n + 1) if n % q == 0]:
            lay = m.build_group_layout(n, p)
            for s in (1, 2, 4):
                gf = oracle.random_f32(s * n * 13, -1.0, 1.0, n * 1000 + p * 10 + s).reshape(s, n, 13)
                th = m.make_sync_states(eng, lay, 13, s, "f32")
                for t in range(s):
                    m.two_hop_micro_step(eng, lay, th, list(gf[t]))
                m.two_hop_boundary(eng, lay, th)
                want = arr[f"acc2/f32/{n}/{p}/{s}/two_hop"]
                for r in range(n):
                    assert np.array_equal(u32(th.shard(r)), u32(want[r])), (n, p, s, r)
                th.close()


def test_events_state_machine_and_confinement(m, engines, oracle, golden):
    arr, dig = golden
    eng = engines(8)
    lay = m.build_group_layout(8, 4)
    g = oracle.random_i64(2 * 8 * 16, -5, 5, 1).reshape(2, 8, 16)
    st = m.make_sync_states(eng, lay, 16, 2, "i64")
    log = []
    eng.clear_traffic()
    for t in range(2):
        m.two_hop_micro_step(eng, lay, st, list(g[t]), log)
    m.two_hop_boundary(eng, lay, st, log)
    got = np.array([[e.step, int(e.phase), e.group_id, e.bytes] for e in log])
    assert np.array_equal(got, arr["sched/events_two_hop"])
    assert eng.traffic() == {(a, b): c for a, b, c in dig["sched/events_traffic"]}
    # micro-steps stay inside partition groups (test_sync_schedule.cpp:134-150)
    eng.clear_traffic()
    st1 = m.make_sync_states(eng, lay, 12, 1, "i64")
    m.two_hop_micro_step(eng, lay, st1, [np.ones(12, np.int64)] * 8)
    assert all(a // 4 == b // 4 for a, b in eng.traffic())
    # state machine (test_sync_schedule.cpp:117-132; golden codes from the reference)
    e4 = engines(4)
    lay2 = m.build_group_layout(4, 2)
    sm = m.make_sync_states(e4, lay2, 8, 2, "i64")
    grads = [np.ones(8, np.int64)] * 4
    codes = []
    for op in "bmbmmbm":
        try:
            (m.two_hop_micro_step(e4, lay2, sm, grads) if op == "m" else m.two_hop_boundary(e4, lay2, sm))
            codes.append(0)
        except m.Error as e:
            codes.append(int(e.code))
    assert codes == arr["sched/state_machine"].tolist()


# ------------------------------------------------------------------ fused paths beyond the reference
def test_bf16_cast_scale_and_zero_accum(m, engines, oracle):
    """K2 fused with bf16->fp32 cast and a power-of-two scale (exact), ZERO_ACCUM vs ACCUMULATE."""
    from paper_2205_00119_b200.collectives import RS_ACCUMULATE, RS_ZERO_ACCUM, reduce_scatter_device
    eng = engines(8)
    p, chunk = 4, 70_001
    buf = eng.alloc(p * chunk * 2)
    out = eng.alloc(chunk * 4)
    vals = []
    for r in range(p):
        eng.generate(buf, r, p * chunk, "bf16", seed=9, step=0, layer=3)
        vals.append(oracle.gen_bf16(9, r, 0, 3, 0, p * chunk))
    ranks = list(range(p))
    ptr_in = [eng.ptr(buf, r) for r in ranks]
    ptr_out = [eng.ptr(out, r) for r in ranks]
    neg0 = np.full(chunk, -0.0, np.float32)
    for r in ranks:
        eng.h2d(out, r, neg0)
    reduce_scatter_device(eng, ranks, ptr_in, p * chunk, ptr_out, "bf16", "f32", 0.25, RS_ZERO_ACCUM)
    reduce_scatter_device(eng, ranks, ptr_in, p * chunk, ptr_out, "bf16", "f32", 0.25, RS_ACCUMULATE,
                          valid_elems=p * chunk - 1000)
    eng.synchronize()
    f = [(v.astype(np.uint32) << 16).view(np.float32) for v in vals]
    for j in ranks:
        sl = slice(j * chunk, (j + 1) * chunk)
        fold = f[0][sl].copy()
        for i in range(1, p):
            fold = fold + f[i][sl]
        first = np.float32(0) + fold * np.float32(0.25)
        idx = np.arange(j * chunk, (j + 1) * chunk)
        fold2 = np.where(idx < p * chunk - 1000, fold, np.float32(0))
        want = first + fold2 * np.float32(0.25)
        assert np.array_equal(u32(eng.d2h(out, j, chunk, "f32")), u32(want)), j


def test_generator_matches_oracle(m, engines, oracle):
    eng = engines(8)
    b = eng.alloc(1 << 22)
    eng.generate(b, 3, 100_003, "f32", seed=77, step=2, layer=5, start=12345)
    assert np.array_equal(u32(eng.d2h(b, 3, 100_003, "f32")), u32(oracle.gen_f32(77, 3, 2, 5, 12345, 100_003)))
    eng.generate(b, 1, 100_003, "bf16", seed=77, step=2, layer=5)
    assert np.array_equal(eng.d2h(b, 1, 100_003, "bf16"), oracle.gen_bf16(77, 1, 2, 5, 0, 100_003))


@pytest.mark.parametrize("wd,length", [(0.0, 300_001), (0.01, 300_001), (0.01, 2_000_003)])
def test_boundary_fused_adam_bitexact(m, engines, oracle, wd, length):
    """Boundary AR's all-gather fused with Adam (K5), bit-exact vs the C restatement."""
    from paper_2205_00119_b200.sync_schedule import AdamConfig, make_adam
    n, p, s = 8, 2, 2
    eng = engines(n)
    lay = m.build_group_layout(n, p)
    g = oracle.random_f32(s * n * length, -1.0, 1.0, 5).reshape(s, n, length)
    st = m.make_sync_states(eng, lay, length, s, "f32")
    for t in range(s):
        m.two_hop_micro_step(eng, lay, st, list(g[t]))
    c = st.shard_elems
    bufs = [eng.alloc(4 * c) for _ in range(3)]
    pb = eng.alloc(2 * c)
    rng = np.random.default_rng(1)
    p0, m0 = rng.standard_normal(c).astype(np.float32), rng.standard_normal(c).astype(np.float32) * 0.01
    v0 = np.abs(rng.standard_normal(c).astype(np.float32)) * 1e-4
    for r in range(n):
        eng.h2d(bufs[0], r, p0)
        eng.h2d(bufs[1], r, m0)
        eng.h2d(bufs[2], r, v0)
    cfg = AdamConfig(lr=3e-4, weight_decay=wd, step=7, grad_scale=1.0 / (n * s))
    m.two_hop_boundary(eng, lay, st, adam=make_adam(st, cfg, *bufs, param_bf16=pb))
    eng.synchronize()
    red, _, _ = oracle.two_hop(g, n, p, "f32")
    for r in range(n):
        wp, wm, wv, wb = oracle.adam(p0, m0, v0, red[r], 3e-4, 0.9, 0.999, 1e-8, wd, 7, 1.0 / (n * s), True)
        assert np.array_equal(u32(eng.d2h(bufs[0], r, c)), u32(wp)), r
        assert np.array_equal(u32(eng.d2h(bufs[1], r, c)), u32(wm)), r
        assert np.array_equal(u32(eng.d2h(bufs[2], r, c)), u32(wv)), r
        assert np.array_equal(eng.d2h(pb, r, c, "bf16"), wb), r
    # and within 1e-6 relative of torch.optim.Adam semantics (fp32)
    import torch
    pt = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([pt], lr=3e-4, weight_decay=wd)
    st_ = opt.state[pt]
    st_["step"] = torch.tensor(6.0)
    st_["exp_avg"] = torch.tensor(m0.copy())
    st_["exp_avg_sq"] = torch.tensor(v0.copy())
    pt.grad = torch.tensor(red[0] * np.float32(1.0 / (n * s)))
    opt.step()
    got = eng.d2h(bufs[0], 0, c)
    ref = pt.detach().numpy()
    assert np.all(np.abs(got - ref) <= 1e-6 * np.maximum(1.0, np.abs(ref)))
