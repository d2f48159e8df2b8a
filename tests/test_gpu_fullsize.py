"""Full-size parity (BASELINE.json C3: BERT-large-shaped 334,088,192 parameters, n=8,
p=2, s=4, fp32 gradients) through properties that do not need the whole job on the
CPU.  The gradients come from the counter-based generator (K6), so the CPU can
evaluate any element of any rank's gradient directly; for a random sample of shard
elements it replays the 2-hop folds (reduce-scatter over the partition group per
micro-step, accumulation over micro-steps, boundary fold over the replication group)
and Adam, and the device result must match BIT-EXACTLY.  Same for the gathered
bf16 parameters (all-gather = concatenation of the group's shards)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def check_sampled(oracle, eng, step, wl, opts, ranks, nsamples=400, seed=7):
    """Bit-exact check of sampled shard elements of `ranks` after one step (see module doc)."""
    n, p, s = wl.n, wl.p, wl.s
    info, segs = step.sync_info()
    S = info.shard_elems
    b = step.buffers()
    rng = np.random.default_rng(seed)
    samples = np.sort(rng.choice(S, nsamples, replace=False))
    # include both ends and every layer boundary
    samples = np.unique(np.concatenate([samples, [0, S - 1]] + [[so, so + c - 1] for _, c, so, _ in segs]))
    seg_of = np.searchsorted([so for _, _, so, _ in segs], samples, side="right") - 1
    seed_m = opts.seed ^ 0x5EED
    for x, q in zip(samples, seg_of):
        ln, c, so, go = segs[q]
        e = int(x - so)
        for r in ranks:
            j = r % p
            members = []  # accumulated gradient of every replication-group member (j, j+p, ...)
            for gg in range(n // p):
                acc = np.float32(0)
                for t in range(s):
                    gi = go + j * c + e
                    if j * c + e < ln:  # partition-group fold, ascending position
                        f = oracle.gen_f32(opts.seed, gg * p + 0, t, 0, gi, 1)[0]
                        for i in range(1, p):
                            f = np.float32(f + oracle.gen_f32(opts.seed, gg * p + i, t, 0, gi, 1)[0])
                    else:
                        f = np.float32(0)
                    acc = np.float32(acc + f) if t else np.float32(np.float32(0) + f)
                members.append(acc)
            red = members[0]
            for a_ in members[1:]:
                red = np.float32(red + a_)
            p0 = oracle.gen_f32(seed_m, j, 0, 255, int(x), 1)
            wp, _, _, wb = oracle.adam(p0, np.zeros(1), np.zeros(1), np.array([red], np.float32), opts.lr, opts.beta1,
                                       opts.beta2, opts.eps, opts.weight_decay, 1, 1.0 / (n * s), want_bf16=True)
            got = eng.d2h(b["master"], r, 1, off=int(x) * 4)
            assert got.view(np.uint32)[0] == wp.view(np.uint32)[0], (int(x), r)
            assert eng.d2h(b["param_bf16"], r, 1, "bf16", off=int(x) * 2)[0] == wb[0], (int(x), r)
    # all-gather: the last gathers of the backward pass (layers 2, 1, 0) left layer l in
    # slot l mod gather_slots (csrc/step.cpp) = the group's pre-update bf16 shards;
    # they ran as one PDL chain, so this also checks that no earlier gather of a slot
    # landed after the last one
    half, slots = step.stats().gather_slot_bytes, step.stats().gather_slots
    for l in range(min(3, len(segs))):
        _, cl, sol, _ = segs[l]
        for pos_e in rng.choice(p * cl, 100, replace=False):
            pos, e = divmod(int(pos_e), cl)
            want = oracle.f32_to_bf16(oracle.gen_f32(seed_m, pos, 0, 255, sol + e, 1))[0]
            for r in ranks[:2]:
                got = eng.d2h(b["gathered"], r, 1, "bf16", off=(l % slots) * half + int(pos_e) * 2)[0]
                assert got == want, (l, r, pos, e)


def test_c3_full_size_sampled_bitexact(oracle):
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, workloads
    import bench
    wl = workloads()["C3"]
    opts = StepOptions(seed=2205, lr=1e-4)
    eng = Engine(n_ranks=wl.n, device=0, arena_bytes=bench.arena_bytes(wl, wl.n, True, wl.n))
    step = MicsStep(eng, wl, opts)
    assert sum(ln for ln, _, _, _ in step.sync_info()[1]) == 334_088_192
    step.run(1)
    eng.synchronize()
    check_sampled(oracle, eng, step, wl, opts, list(range(wl.n)))
    step.close()
    eng.close()


@pytest.mark.parametrize("path", ["k8", "k9"])
def test_c3_full_size_every_element_bitexact(oracle, monkeypatch, path):
    """C3 at full size (334,088,192 parameters, n=8, p=2, s=4) on one GPU, EVERY shard
    element of every rank: the device's master / bf16 (and m / v of two ranks) after one
    step equal the oracle's whole-shard step (ora_step1_shard: the generator's
    gradients folded in the reference's order, then Adam), bit for bit.  k8: the default
    fused tail; k9: the overlapped tail with the fused layer-group boundary forced on one
    GPU."""
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, workloads
    import bench
    if path == "k9":
        monkeypatch.setenv("MICS_FUSED_TAIL", "0")
        monkeypatch.setenv("MICS_TAIL_OVERLAP", "1")
        monkeypatch.setenv("MICS_TAIL_FUSED", "1")
    wl = workloads()["C3"]
    opts = StepOptions(seed=2205, lr=1e-4)
    eng = Engine(n_ranks=wl.n, device=0, arena_bytes=bench.arena_bytes(wl, wl.n, True, wl.n))
    step = MicsStep(eng, wl, opts)
    info, segs = step.sync_info()
    S = info.shard_elems
    step.run(1)
    eng.synchronize()
    b = step.buffers()
    for j in range(wl.p):
        master, m, v, bf = oracle.step1_shard(opts.seed, wl.n, wl.p, wl.s, j, segs, S, opts.lr, opts.beta1,
                                              opts.beta2, opts.eps, opts.weight_decay)
        for r in range(j, wl.n, wl.p):
            got = eng.d2h(b["master"], r, S)
            bad = np.flatnonzero(got.view(np.uint32) != master.view(np.uint32))
            assert bad.size == 0, (r, bad[:5], bad.size)
            assert np.array_equal(eng.d2h(b["param_bf16"], r, S, "bf16"), bf), r
        r = j  # the optimizer state of one replica per position
        assert np.array_equal(eng.d2h(b["exp_avg"], r, S).view(np.uint32), m.view(np.uint32))
        assert np.array_equal(eng.d2h(b["exp_avg_sq"], r, S).view(np.uint32), v.view(np.uint32))
    step.close()
    eng.close()
