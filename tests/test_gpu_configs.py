"""Config-level parity: every BASELINE.json config at its own
shapes, on the GPU, against the reference or its pinned restatement.

* C1 (4-layer MLP, 4,198,400 params, n=8, p=2, s=4): the 2-hop and alternative
  schedules over the whole gradient (one segment) with the reference's generator
  (mt19937(2205) U(-1,1)) — per-rank digests of the shards equal the digests the
  UNMODIFIED reference produced (tests/golden/make_golden.py, "cfg/c1_full/*"),
  acceptance_main.cpp:93-152 / sync_schedule.hpp:118-232 at full size; and the step
  driver on C1's 4 x 1,049,600 layers against the CPU restatement of the whole step.
* C4 (GPT-2 1.5B, 1,557,608,000 params, bf16 gradients generated in-step): the
  hierarchical all-gather at the SURVEY's non-degenerate shapes (k=2 with p=4;
  p=8 with k=4; collectives.cpp:192-291), full size, sampled bit-exact shards and
  every gathered slot.
* C5 (BERT-10B shapes): the embedding plus one 78,676,480-parameter block at p=8
  (ZeRO-3) and p=4, bf16 gradients generated in-step (K6), sampled bit-exact.
* C2 (collective sweep): one 1 GiB all-gather and one 1 GiB reduce-scatter at p=8
  against the oracle, every output bit-compared.
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def bf16_to_f32(b):
    return (np.asarray(b).astype(np.uint32) << 16).view(np.float32)


@pytest.fixture(scope="module")
def m():
    import paper_2205_00119_b200 as m
    return m


# ------------------------------------------------------------------ C1
@pytest.mark.parametrize("mode", ["two_hop", "alternative"])
def test_c1_full_size_schedule_equals_reference(m, oracle, golden, mode):
    arr, dig = golden
    n, p, s, length = 8, 2, 4, 4_198_400
    g = oracle.random_f32(s * n * length, -1.0, 1.0, 2205).reshape(s, n, length)
    eng = m.Engine(n_ranks=n, device=0, arena_bytes=1 << 30)
    lay = m.build_group_layout(n, p)
    st = m.make_sync_states(eng, lay, length, s, "f32")
    for t in range(s):
        if mode == "two_hop":
            m.two_hop_micro_step(eng, lay, st, list(g[t]))
        else:
            m.alternative_schedule_step(eng, lay, st, list(g[t]))
    if mode == "two_hop":
        m.two_hop_boundary(eng, lay, st)
    else:
        m.alternative_boundary(st)
    shards = np.stack(st.shards())[:, :(length + p - 1) // p]
    assert [digest(x) for x in shards] == dig[f"cfg/c1_full/{mode}"]
    assert np.array_equal(u32(shards[:, ::9973]), u32(arr[f"cfg/c1_full/{mode}_every_9973"]))
    st.close()
    eng.close()


def test_c1_step_full_size(oracle):
    """The step driver on C1 itself (4 x 1,049,600 layers, n=8, p=2, s=4): parameters,
    Adam state and bf16 copies of every rank against the CPU restatement of the step."""
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, workloads
    from test_gpu_step import expected_step
    wl = workloads()["C1"]
    assert wl.params == 4_198_400
    opts = StepOptions(seed=2205, lr=1e-3, weight_decay=0.01)
    eng = Engine(n_ranks=wl.n, device=0, arena_bytes=1 << 30)
    step = MicsStep(eng, wl, opts)
    info, segs = step.sync_info()
    b = step.buffers()
    S = info.shard_elems
    step.run(1)
    eng.synchronize()
    want, _ = expected_step(oracle, wl.n, wl.p, wl.s, segs, "f32", opts.seed, False, opts)
    for r in range(wl.n):
        wp, wm, wv, wb = want[r]
        assert np.array_equal(u32(eng.d2h(b["master"], r, S)), u32(wp)), r
        assert np.array_equal(u32(eng.d2h(b["exp_avg"], r, S)), u32(wm)), r
        assert np.array_equal(u32(eng.d2h(b["exp_avg_sq"], r, S)), u32(wv)), r
        assert np.array_equal(eng.d2h(b["param_bf16"], r, S, "bf16"), wb), r
    step.close()
    eng.close()


# ------------------------------------------------------------------ C4 / C5 (full-size shapes, sampled)
def check_step_sampled(oracle, eng, step, wl, opts, nsamples=300, seed=7):
    """One step of `wl` on `eng` with gradients from the counter-based generator (K6,
    f32 or bf16), checked BIT-EXACTLY at sampled shard elements of every rank (both
    ends and every layer boundary included) by replaying the folds and Adam on the
    CPU, and every gathered slot (the last backward gathers left layer l in slot
    l mod gather_slots) at sampled positions against the group's pre-update bf16 shards."""
    n, p, s = wl.n, wl.p, wl.s
    info, segs = step.sync_info()
    S = info.shard_elems
    b = step.buffers()
    rng = np.random.default_rng(seed)
    samples = np.sort(rng.choice(S, nsamples, replace=False))
    samples = np.unique(np.concatenate([samples, [0, S - 1]] + [[so, so + c - 1] for _, c, so, _ in segs]))
    seg_of = np.searchsorted([so for _, _, so, _ in segs], samples, side="right") - 1
    seed_m = opts.seed ^ 0x5EED

    def grad(rank, t, gi):
        if wl.grad_dtype == "bf16":
            return bf16_to_f32(oracle.gen_bf16(opts.seed, rank, t, 0, gi, 1))[0]
        return oracle.gen_f32(opts.seed, rank, t, 0, gi, 1)[0]

    for x, q in zip(samples, seg_of):
        ln, c, so, go = segs[q]
        e = int(x - so)
        for j in range(p):  # every replica of position j ends with the same parameters
            members = []
            for gg in range(n // p):
                acc = np.float32(0)
                for t in range(s):
                    if j * c + e < ln:  # partition-group fold, ascending position
                        f = grad(gg * p, t, go + j * c + e)
                        for i in range(1, p):
                            f = np.float32(f + grad(gg * p + i, t, go + j * c + e))
                    else:
                        f = np.float32(0)
                    acc = np.float32(acc + f) if t else np.float32(np.float32(0) + f)
                members.append(acc)
            red = members[0]
            for a_ in members[1:]:  # boundary fold over the replication group, ascending
                red = np.float32(red + a_)
            p0 = oracle.gen_f32(seed_m, j, 0, 255, int(x), 1)
            wp, wm, wv, wb = oracle.adam(p0, np.zeros(1), np.zeros(1), np.array([red], np.float32), opts.lr,
                                         opts.beta1, opts.beta2, opts.eps, opts.weight_decay, 1, 1.0 / (n * s),
                                         want_bf16=True)
            for r in range(j, n, p):
                assert eng.d2h(b["master"], r, 1, off=int(x) * 4).view(np.uint32)[0] == u32(wp)[0], (int(x), r)
                assert eng.d2h(b["exp_avg_sq"], r, 1, off=int(x) * 4).view(np.uint32)[0] == u32(wv)[0], (int(x), r)
                assert eng.d2h(b["param_bf16"], r, 1, "bf16", off=int(x) * 2)[0] == wb[0], (int(x), r)
    half, slots = step.stats().gather_slot_bytes, step.stats().gather_slots
    for l in range(min(3, len(segs))):
        _, cl, sol, _ = segs[l]
        for pos_e in rng.choice(p * cl, 64, replace=False):
            pos, e = divmod(int(pos_e), cl)
            want = oracle.f32_to_bf16(oracle.gen_f32(seed_m, pos, 0, 255, sol + e, 1))[0]
            for r in range(n):
                got = eng.d2h(b["gathered"], r, 1, "bf16", off=(l % slots) * half + int(pos_e) * 2)[0]
                assert got == want, (l, r, pos, e)
        # both ends of every slot, every position
        for pos in range(p):
            for e in (0, cl - 1):
                want = oracle.f32_to_bf16(oracle.gen_f32(seed_m, pos, 0, 255, sol + e, 1))[0]
                for r in range(n):
                    got = eng.d2h(b["gathered"], r, 1, "bf16", off=(l % slots) * half + (pos * cl + e) * 2)[0]
                    assert got == want, (l, r, pos, e)


def run_sampled(oracle, wl, expect_params):
    import bench
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions
    assert wl.params == expect_params
    opts = StepOptions(resident_grads=False, seed=2205, lr=1e-4)
    eng = Engine(n_ranks=wl.n, device=0, arena_bytes=bench.arena_bytes(wl, wl.n, False, wl.n))
    step = MicsStep(eng, wl, opts)
    step.run(1)
    eng.synchronize()
    check_step_sampled(oracle, eng, step, wl, opts)
    stats = step.stats()
    step.close()
    eng.close()
    return stats


@pytest.mark.parametrize("p,k", [(4, 2), (8, 4)])
def test_c4_hierarchical_full_size_sampled(oracle, p, k):
    """GPT-2 1.5B (h1600, i6400, L48, V50257, l1024) with the hierarchical all-gather at
    the shapes that exercise all three stages (the literal 2 x 4 layout is
    degenerate): ceil(2L/3)+1 merged k_hier launches per micro-step, bf16 in-step gradients."""
    import dataclasses

    from paper_2205_00119_b200.workloads import workloads
    wl = dataclasses.replace(workloads()["C4"], p=p, hier_k=k)
    stats = run_sampled(oracle, wl, 1_557_608_000)
    assert stats.ag_launches == wl.s * (-(-2 * len(wl.layer_params) // 3) + 1)


@pytest.mark.parametrize("p", [8, 4])
def test_c5_shapes_sampled(oracle, p):
    """BERT-10B shapes (h2560, i10240, V32008, l512): the 83,251,200-parameter embedding
    and one 78,676,480-parameter block, p=8 (ZeRO-3) and p=4, bf16 in-step gradients."""
    from paper_2205_00119_b200.workloads import Workload, workloads
    c5 = workloads()["C5p8"]
    assert c5.layer_params[0] == 83_251_200 and c5.layer_params[1] == 78_676_480 and c5.params == 10_075_164_160
    wl = Workload(f"C5 shapes p={p}", c5.layer_params[:2], p=p, s=c5.s, grad_dtype="bf16")
    run_sampled(oracle, wl, 83_251_200 + 78_676_480)


# ------------------------------------------------------------------ C2 at 1 GiB
def test_c2_one_gib_all_gather_and_reduce_scatter(m, oracle):
    """C2's largest point, p=8: a 1 GiB all-gather (128 MiB chunks) and a 1 GiB fp32
    reduce-scatter (256M elements per rank) — every output compared with the oracle."""
    from paper_2205_00119_b200.collectives import all_gather_device, reduce_scatter_device
    p = 8
    M = 1 << 30
    chunk = M // p
    eng = m.Engine(n_ranks=p, device=0, arena_bytes=10 << 30)
    ranks = list(range(p))
    # all-gather: random bytes, expected output = the oracle's gather (concatenation)
    rng = np.random.default_rng(2205)
    shards = rng.integers(0, 256, (p, chunk), dtype=np.uint8)
    mark = eng.mark()
    src, out = eng.alloc(chunk), eng.alloc(M)
    for r in ranks:
        eng.h2d(src, r, shards[r])
    all_gather_device(eng, ranks, [eng.ptr(src, r) for r in ranks], chunk, [eng.ptr(out, r) for r in ranks])
    eng.synchronize()
    want = oracle.all_gather(shards[:, :4096])[0]  # the restatement on a prefix of every chunk
    assert np.array_equal(want, np.concatenate([s[:4096] for s in shards]))
    flat = shards.reshape(-1)
    for r in ranks:
        got = eng.d2h(out, r, M, "u8")
        assert np.array_equal(got, flat), r
        if r == 0:
            assert digest(got) == digest(flat)
    del flat, shards
    eng.release(mark)
    # reduce-scatter: fp32 inputs from the counter-based generator on both sides
    elems = M // 4
    inp, res = eng.alloc(M), eng.alloc(M // p)
    for r in ranks:
        eng.generate(inp, r, elems, "f32", seed=2205, step=0, layer=7)
    reduce_scatter_device(eng, ranks, [eng.ptr(inp, r) for r in ranks], elems, [eng.ptr(res, r) for r in ranks])
    host = np.stack([oracle.gen_f32(2205, r, 0, 7, 0, elems) for r in ranks])
    want = oracle.reduce_scatter(host, "f32")
    del host
    eng.synchronize()
    for r in ranks:
        got = eng.d2h(res, r, elems // p)
        assert np.array_equal(u32(got), u32(want[r])), r
    eng.close()
