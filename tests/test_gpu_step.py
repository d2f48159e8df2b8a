"""GPU parity of the MiCS step driver (csrc/step.cpp) against a restatement of the
step on the CPU: per-layer all-gathers, s micro-step reduce-scatters with the
pinned fold order, the boundary replication-group fold and the documented Adam —
bit-exact, for the 2-hop schedule, the alternative (global all-reduce) schedule,
bf16 gradients and the hierarchical all-gather.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def bf16_to_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def expected_step(oracle, n, p, s, segs, grad_dtype, seed, alternative, opts):
    """Returns per-rank (master, m, v, param_bf16) after one step, and the initial bf16 params."""
    S = sum(c for _, c, _, _ in segs)
    G = sum(p * c for _, c, _, _ in segs)
    grads = np.zeros((s, n, G), np.float32)
    for t in range(s):
        for r in range(n):
            if grad_dtype == "bf16":
                grads[t, r] = bf16_to_f32(oracle.gen_bf16(seed, r, t, 0, 0, G))
            else:
                grads[t, r] = oracle.gen_f32(seed, r, t, 0, 0, G)
    acc = np.zeros((n, S), np.float32)
    for r in range(n):
        j, g = r % p, r // p
        for t in range(s):
            fold = np.zeros(S, np.float32)
            for ln, c, so, go in segs:
                e = np.arange(c)
                valid = (j * c + e) < ln
                if alternative:  # all-reduce over all n ranks, ascending rank
                    f = grads[t, 0, go + j * c + e].copy()
                    for i in range(1, n):
                        f = f + grads[t, i, go + j * c + e]
                else:  # reduce-scatter in the partition group, ascending position
                    f = grads[t, g * p + 0, go + j * c + e].copy()
                    for i in range(1, p):
                        f = f + grads[t, g * p + i, go + j * c + e]
                fold[so:so + c] = np.where(valid, f, np.float32(0))
            acc[r] = (np.float32(0) + fold) if t == 0 else (acc[r] + fold)
    red = np.zeros_like(acc)
    for r in range(n):
        if alternative:
            red[r] = acc[r]
        else:  # boundary all-reduce in the replication group, ascending position
            j = r % p
            f = acc[j].copy()
            for q in range(1, n // p):
                f = f + acc[j + q * p]
            red[r] = f
    out, init = [], []
    for r in range(n):
        m0 = oracle.gen_f32(seed ^ 0x5EED, r % p, 0, 255, 0, S)
        init.append(m0)
        out.append(oracle.adam(m0, np.zeros(S), np.zeros(S), red[r], opts.lr, opts.beta1, opts.beta2, opts.eps,
                               opts.weight_decay, 1, 1.0 / (n * s), want_bf16=True))
    return out, init


@pytest.mark.parametrize("alternative,grad_dtype,hier_k,p", [
    (False, "f32", 0, 2), (True, "f32", 0, 2), (False, "bf16", 0, 4), (False, "f32", 2, 4), (True, "bf16", 0, 8)])
def test_step_matches_cpu_restatement(oracle, alternative, grad_dtype, hier_k, p):
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    n, s = 8, 3
    layers = [10_000, 4_099, 777, 65_536]
    wl = Workload("test", layers, p=p, s=s, grad_dtype=grad_dtype, hier_k=hier_k)
    opts = StepOptions(resident_grads=not alternative, alternative=alternative, seed=77, lr=1e-3, weight_decay=0.01)
    eng = Engine(n_ranks=n, device=0, arena_bytes=256 << 20)
    step = MicsStep(eng, wl, opts)
    info, segs = step.sync_info()
    bufs = step.buffers()
    S = info.shard_elems
    step.run(1)
    eng.synchronize()
    want, init = expected_step(oracle, n, p, s, segs, grad_dtype, 77, alternative, opts)
    for r in range(n):
        wp, wm, wv, wb = want[r]
        assert np.array_equal(u32(eng.d2h(bufs["master"], r, S)), u32(wp)), r
        assert np.array_equal(u32(eng.d2h(bufs["exp_avg"], r, S)), u32(wm)), r
        assert np.array_equal(u32(eng.d2h(bufs["exp_avg_sq"], r, S)), u32(wv)), r
        assert np.array_equal(eng.d2h(bufs["param_bf16"], r, S, "bf16"), wb), r
    # the last gathers (backward pass, layers 2, 1, 0) left layer l in slot l mod 3
    # (csrc/step.cpp gather_slots): the pre-update bf16 params of the group
    stats = step.stats()
    half, slots = stats.gather_slot_bytes, stats.gather_slots
    for l in range(min(3, len(segs))):
        _, cl, sol, _ = segs[l]
        for r in range(n):
            g = r // p
            got = eng.d2h(bufs["gathered"], r, p * cl, "bf16", off=(l % slots) * half)
            for i in range(p):
                want_bf = oracle.f32_to_bf16(init[g * p + i][sol:sol + cl])
                assert np.array_equal(got[i * cl:(i + 1) * cl], want_bf), (l, r, i)
    # flat: one k_copy launch per layer visit; hierarchical: ceil(2L/3)+1 merged k_hier
    # launches per micro-step (launch y = stage 1 of 3 visits + stage 3 of the 3 before)
    want_ag = s * (-(-2 * len(layers) // 3) + 1) if hier_k and p > hier_k else 2 * s * len(layers)
    assert stats.launches > 0 and stats.ag_launches == want_ag
    step.close()
    eng.close()


@pytest.mark.parametrize("graph", ["1", "0"])
def test_hier_merged_matches_per_visit(monkeypatch, graph):
    """The comm-only step's merged hierarchical launches (launch y = stage 1 of G visits +
    stage 3 of the previous G, done counters instead of barriers; G = 3, 1, 4) vs one
    k_hier launch per visit (MICS_HIER_MERGE=0): same parameters and gathered layers
    over three steps, at p=4/k=2 and p=8/k=4, with the default grid and a 5-CTA cap."""
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_GRAPH", graph)
    for p, k in ((4, 2), (8, 4)):
        res = []
        for merge, visits, cap in (("0", "3", 0), ("1", "3", 0), ("1", "1", 0), ("1", "4", 0), ("1", "3", 5)):
            monkeypatch.setenv("MICS_HIER_MERGE", merge)
            monkeypatch.setenv("MICS_HIER_VISITS", visits)
            eng = Engine(n_ranks=8, device=0, arena_bytes=256 << 20)
            eng.set_parallelism(0, cap)
            wl = Workload("hm", [70_000, 12_345, 40_000, 9_999, 33_333, 4_096], p=p, s=2, grad_dtype="bf16", hier_k=k)
            step = MicsStep(eng, wl, StepOptions(seed=29))
            step.run(3)
            eng.synchronize()
            b, (info, segs) = step.buffers(), step.sync_info()
            half, slots = step.stats().gather_slot_bytes, step.stats().gather_slots
            res.append([(u32(eng.d2h(b["master"], r, info.shard_elems)),) +
                        tuple(eng.d2h(b["gathered"], r, p * segs[l][1], "bf16", off=(l % slots) * half)
                              for l in range(3)) for r in range(8)])
            step.close()
            eng.close()
        for other in res[1:]:
            for r in range(8):
                for a, c in zip(res[0][r], other[r]):
                    assert np.array_equal(a, c), (p, k, r)


def test_step_two_steps_deterministic(oracle):
    """Two steps, twice: identical bits (the step is deterministic and replayable)."""
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    wl = Workload("det", [50_000, 12_345], p=2, s=2)
    res = []
    for _ in range(2):
        eng = Engine(n_ranks=8, device=0, arena_bytes=128 << 20)
        step = MicsStep(eng, wl, StepOptions(seed=5))
        step.run(2)
        eng.synchronize()
        res.append(eng.d2h(step.buffers()["master"], 3, step.sync_info()[0].shard_elems))
        step.close()
        eng.close()
    assert np.array_equal(u32(res[0]), u32(res[1]))


@pytest.mark.parametrize("fused_tail", ["0", "1"])
def test_graph_replay_matches_eager(monkeypatch, fused_tail):
    """The CUDA-graph replayed step (default) gives the same bits as enqueueing every
    kernel per step, across replays, an interleaved profiled (eager) step and the
    per-step Adam scalars it reads from device memory (two-kernel boundary or K8)."""
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_FUSED_TAIL", fused_tail)
    wl = Workload("graph", [70_000, 12_345, 40_000, 9_999], p=2, s=2)
    res = {}
    for graph in ("0", "1"):
        monkeypatch.setenv("MICS_GRAPH", graph)
        eng = Engine(n_ranks=8, device=0, arena_bytes=256 << 20)
        step = MicsStep(eng, wl, StepOptions(seed=21, lr=1e-3, weight_decay=0.01))
        l0 = eng.launches
        step.run(2)
        step.profile()
        step.run(2)
        eng.synchronize()
        assert step.stats().adam_step == 5
        if graph == "1":  # replays count every captured kernel (+ the scalar update)
            assert eng.launches - l0 >= 5 * step.stats().launches
        S = step.sync_info()[0].shard_elems
        b = step.buffers()
        res[graph] = [eng.d2h(b[k], r, S) for k in ("master", "exp_avg", "exp_avg_sq") for r in range(8)]
        res[graph].append(eng.d2h(b["param_bf16"], 3, S, "bf16"))
        step.close()
        eng.close()
    for x, y in zip(res["0"], res["1"]):
        assert np.array_equal(x.view(np.uint16), y.view(np.uint16))


@pytest.mark.parametrize("resident", [True, False])
def test_run_host_matches_device_resident(resident):
    """e2e path (H2D on a copy stream, overlapping the gathers): same bits as the
    step run on the same gradients already resident in HBM."""
    from paper_2205_00119_b200.engine import Engine, host_alloc, host_free
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    wl = Workload("host", [30_000, 12_345, 20_000], p=2, s=3)
    eng = Engine(n_ranks=8, device=0, arena_bytes=256 << 20)
    step = MicsStep(eng, wl, StepOptions(seed=3, lr=1e-3, resident_grads=resident))
    G = step.stats().grad_elems
    host, hptr = host_alloc(G * 4)
    g = np.random.default_rng(7).uniform(-1, 1, G).astype(np.float32)
    host[:] = g.view(np.uint8)
    res, rptr = host_alloc(8 * 4096 * 4)
    step.run_host(hptr, 2, rptr)
    eng.synchronize()
    S = step.sync_info()[0].shard_elems
    got = [eng.d2h(step.buffers()["master"], r, S) for r in range(8)]
    assert np.array_equal(res[:min(4096, S) * 4].view(np.float32), got[0][:min(4096, S)])
    step.close()
    # reference: the same gradients placed in every slot, then the device-resident step
    step2 = MicsStep(eng, wl, StepOptions(seed=3, lr=1e-3, resident_grads=True))
    b = step2.buffers()
    for r in range(8):
        for t in range(wl.s):
            eng.h2d(b["grads"], r, g, off=t * G * 4)
    step2.run(2)
    eng.synchronize()
    for r in range(8):
        assert np.array_equal(u32(eng.d2h(b["master"], r, S)), u32(got[r])), r
    step2.close()
    host_free(hptr)
    host_free(rptr)
    eng.close()


@pytest.mark.parametrize("graph", ["1", "0"])
def test_overlapped_tail_matches_in_order(monkeypatch, graph):
    """Overlapped tail (last reduce-scatter per layer group on the main stream, each
    group's boundary all-reduce + Adam on side streams, as two kernels or as the fused
    K9 launch): same bits as the in-order step over several steps, with a profiled
    (serialised) step and a host-input step in between."""
    from paper_2205_00119_b200.engine import Engine, host_alloc, host_free
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_GRAPH", graph)
    monkeypatch.setenv("MICS_FUSED_TAIL", "0")  # the in-order reference path, not K8 (one GPU)
    # the 1.5M / 700k layers give layer groups of several K9 blocks (65,536 elements) per owner
    wl = Workload("tail", [1_500_000, 70_000, 12_345, 700_000, 40_000, 9_999, 33_333, 4_096], p=2, s=3)
    res = {}
    for tail in ("0", "1", "1f"):
        monkeypatch.setenv("MICS_TAIL_OVERLAP", tail[0])
        monkeypatch.setenv("MICS_TAIL_FUSED", "1" if tail == "1f" else "0")
        eng = Engine(n_ranks=8, device=0, arena_bytes=1 << 30)
        step = MicsStep(eng, wl, StepOptions(seed=13, lr=1e-3, weight_decay=0.01))
        G = step.stats().grad_elems
        host, hptr = host_alloc(G * 4)
        host[:] = np.random.default_rng(1).uniform(-1, 1, G).astype(np.float32).view(np.uint8)
        step.run(2)
        prof = step.profile()
        step.run_host(hptr, 1)
        step.run(1)
        eng.synchronize()
        assert prof["boundary_ms"] > 0 and prof["reducescatter_ms"] > 0
        S = step.sync_info()[0].shard_elems
        b = step.buffers()
        res[tail] = [eng.d2h(b[k], r, S) for k in ("master", "exp_avg", "exp_avg_sq") for r in range(8)]
        st = step.stats()
        res[tail + "launch"] = (st.rs_launches, st.bnd_launches, st.rs_hbm_bytes + st.rs_remote_bytes,
                                st.bnd_hbm_bytes + st.bnd_remote_bytes)
        step.close()
        host_free(hptr)
        eng.close()
    for t in ("1", "1f"):
        for x, y in zip(res["0"], res[t]):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), t
        # same reduce-scatter bytes; the tail splits the last reduce-scatter and the boundary per layer group
        assert res[t + "launch"][2] == res["0launch"][2]
        assert res[t + "launch"][0] > res["0launch"][0]
    assert res["1launch"][1] > res["0launch"][1]
    # K9: one boundary launch per layer group (2 groups) instead of two (8 groups); the
    # same boundary bytes
    assert res["1flaunch"][1] < res["1launch"][1]
    assert res["1flaunch"][3] == res["1launch"][3]


@pytest.mark.parametrize("p,s,grad_dtype", [(2, 3, "f32"), (4, 2, "bf16"), (8, 2, "f32"), (2, 1, "bf16")])
def test_fused_tail_matches_unfused(monkeypatch, p, s, grad_dtype):
    """K8 (last reduce-scatter + boundary all-reduce + Adam in one kernel, all ranks on one
    GPU): same bits as the K2 + K2 + K5 sequence over several steps (graph, profiled and
    host-input steps included), for every instantiated (replicas, group size)."""
    from paper_2205_00119_b200.engine import Engine, host_alloc, host_free
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    wl = Workload("ft", [70_000, 12_345, 300_000, 40_000, 9_999, 4_096], p=p, s=s, grad_dtype=grad_dtype)
    res = {}
    for fused in ("0", "1"):
        monkeypatch.setenv("MICS_FUSED_TAIL", fused)
        eng = Engine(n_ranks=8, device=0, arena_bytes=256 << 20)
        step = MicsStep(eng, wl, StepOptions(seed=17, lr=1e-3, weight_decay=0.02))
        G = step.stats().grad_elems
        szg = 2 if grad_dtype == "bf16" else 4
        host, hptr = host_alloc(G * szg)
        host[:] = np.random.default_rng(2).integers(0, 255, G * szg, dtype=np.uint8) & 0x3f
        step.run(2)
        step.profile()
        step.run_host(hptr, 1)
        step.run(1)
        eng.synchronize()
        S = step.sync_info()[0].shard_elems
        b = step.buffers()
        res[fused] = [eng.d2h(b[k], r, S) for k in ("master", "exp_avg", "exp_avg_sq") for r in range(8)]
        res[fused].append(eng.d2h(b["param_bf16"], 6, S, "bf16"))
        step.close()
        host_free(hptr)
        eng.close()
    for x, y in zip(res["0"], res["1"]):
        assert np.array_equal(x.view(np.uint16), y.view(np.uint16))
