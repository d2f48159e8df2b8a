"""One process driving several GPUs (mics_init_devices) — the reference's single
in-process engine (collectives.hpp:42-62) spread over NVLink: virtual ranks
node-major over the GPUs, one member context per GPU, the device flag barriers of a
multi-process job.  The whole API must give the bits of the single-GPU engine and of
the oracle: host-buffer collectives (tests/test_gpu_parity.py runs all of them on two
GPUs too), persistent plans on device pointers, the 2-hop sync, and the step driver."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2205_00119_b200 as m
    return m


def u8(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_group_layout_and_traffic(m, oracle):
    eng = m.Engine(n_ranks=16, arena_bytes=256 << 20, devices=[0, 1])
    assert eng.local_ranks == list(range(16)) and [eng.gpu_of(r) for r in (0, 7, 8, 15)] == [0, 0, 1, 1]
    one = m.Engine(n_ranks=16, device=0, arena_bytes=256 << 20)
    shards = list(oracle.random_shards(16, 9_999, 4))
    cl = m.ClusterSpec(num_nodes=4, devices_per_node=4, intra_node_bandwidth=1, inter_node_bandwidth_per_node=1)
    for e in (eng, one):
        e.clear_traffic()
        out = m.hierarchical_all_gather(e, m.build_group_layout(16, 8), cl, shards)
        assert np.array_equal(np.stack(out), oracle.hier_all_gather(np.stack(shards), 8, 4))
        grp = m.CollectiveGroup([6, 7, 8, 9])  # straddles the two GPUs
        rs = m.reduce_scatter(e, grp, list(oracle.random_f32(4 * 4 * 5000, -1, 1, 3).reshape(4, -1)), "f32")
        assert np.array_equal(u8(np.stack(rs)), u8(oracle.reduce_scatter(
            oracle.random_f32(4 * 4 * 5000, -1, 1, 3).reshape(4, -1), "f32")))
    assert eng.traffic() == one.traffic()
    eng.close()
    one.close()


def test_device_pointer_plans_across_gpus(m, oracle):
    from paper_2205_00119_b200.collectives import RS_STORE, plan_all_gather, plan_reduce_scatter
    eng = m.Engine(n_ranks=8, arena_bytes=256 << 20, devices=[0, 1])
    p, chunk = 8, (1 << 20) + 16
    src, dst = eng.alloc(p * chunk), eng.alloc(p * chunk)
    x = oracle.random_f32(p * p * chunk // 4, -1, 1, 8).reshape(p, -1)
    for r in range(p):
        eng.h2d(src, r, x[r])
    ranks = list(range(p))
    rs = plan_reduce_scatter(eng, ranks, [eng.ptr(src, r) for r in ranks], p * chunk // 4,
                             [eng.ptr(dst, r) for r in ranks], "f32", mode=RS_STORE)
    rs.run(3)
    eng.synchronize()
    want = oracle.reduce_scatter(x, "f32")
    for r in ranks:
        assert np.array_equal(u8(eng.d2h(dst, r, chunk // 4)), u8(want[r])), r
    ag = plan_all_gather(eng, ranks, [eng.ptr(dst, r) for r in ranks], chunk, [eng.ptr(src, r) for r in ranks])
    ag.run(2)
    eng.synchronize()
    flat = u8(want).reshape(-1)
    for r in ranks:
        assert np.array_equal(eng.d2h(src, r, p * chunk, "u8"), flat), r
    rs.close()
    ag.close()
    eng.close()


@pytest.mark.parametrize("p,k,alt,gdt", [(2, 0, False, "f32"), (8, 0, False, "f32"), (4, 0, True, "bf16"),
                                         (8, 4, False, "bf16"), (4, 2, False, "f32")])
def test_step_on_two_gpus_equals_one_gpu(m, p, k, alt, gdt):
    """The step driver with its 8 ranks over two GPUs of one process: the same
    parameters, Adam state and gather slots as on one GPU after two graph-replayed
    steps, an eager profiled step and a host-input step."""
    from paper_2205_00119_b200.engine import host_alloc, host_free
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    wl = Workload("md", [70_000, 12_345, 40_000, 9_999], p=p, s=2, grad_dtype=gdt, hier_k=k)
    res = []
    for devices in (None, [0, 1]):
        eng = m.Engine(n_ranks=8, device=0, arena_bytes=256 << 20, devices=devices)
        step = MicsStep(eng, wl, StepOptions(seed=41, lr=1e-3, resident_grads=not alt, alternative=alt))
        step.run(2)
        step.profile()
        info = step.sync_info()[0]
        ge = info.grad_elems * (2 if gdt == "bf16" else 4)
        host, hptr = host_alloc(ge)
        host[:] = np.random.default_rng(3).integers(0, 255, ge, dtype=np.uint8) & 0x3F  # small finite values
        step.run_host(hptr, 1)
        eng.synchronize()
        b, S = step.buffers(), info.shard_elems
        half, slots = step.stats().gather_slot_bytes, step.stats().gather_slots
        res.append([(u8(eng.d2h(b["master"], r, S)), u8(eng.d2h(b["exp_avg_sq"], r, S)),
                     u8(eng.d2h(b["gathered"], r, slots * half // 2, "bf16"))) for r in range(8)])
        host_free(hptr)
        step.close()
        eng.close()
    for r in range(8):
        for a, c in zip(res[0][r], res[1][r]):
            assert np.array_equal(a, c), r


def test_compute_step_on_two_gpus_equals_one_gpu(m):
    """The step with its layer GEMMs (K7, three streams, copy-engine gathers) with the 8
    ranks over two GPUs of one process: the same parameters and gradients as on one GPU
    (every GEMM tile is computed the same way on either GPU)."""
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    h = 64
    wl = Workload("cmp", [h * 40, h * 37, h * 56], p=2, s=2, hidden=h, micro_batch=8, seq_len=16)
    res = []
    for devices in (None, [0, 1]):
        eng = m.Engine(n_ranks=8, device=0, arena_bytes=256 << 20, devices=devices)
        step = MicsStep(eng, wl, StepOptions(seed=91, lr=1e-3, compute=True))
        step.run(2)
        eng.synchronize()
        info = step.sync_info()[0]
        b = step.buffers()
        res.append([(u8(eng.d2h(b["master"], r, info.shard_elems)), u8(eng.d2h(b["grads"], r, info.grad_elems)))
                    for r in range(8)])
        step.close()
        eng.close()
    for r in range(8):
        for a, c in zip(res[0][r], res[1][r]):
            assert np.array_equal(a, c), r
