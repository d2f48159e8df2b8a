"""Adversarial stress of the relaxed device barrier protocol (kernels.cu bar_entry /
bar_exit; MICS_BAR_STRICT=0, the default) against the fully fenced one
(MICS_BAR_STRICT=1): thousands of back-to-back barrier-carrying launches across two
GPUs — replayed steps whose partition groups and hierarchical gathers span the GPUs,
and chains of accumulate-mode reduce-scatters + all-gathers whose every result feeds
the next launch — must leave bit-identical state.  A stale read anywhere in the chain
would compound into different bits."""
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


def _run(m, monkeypatch, strict, steps, chain):
    from paper_2205_00119_b200.collectives import RS_ACCUMULATE, plan_all_gather, plan_reduce_scatter
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_BAR_STRICT", strict)
    out = []
    for k in (0, 4):  # flat p=8 and hierarchical p=8, k=4: every group spans both GPUs
        eng = m.Engine(n_ranks=8, arena_bytes=128 << 20, devices=[0, 1])
        step = MicsStep(eng, Workload("stress", [9_000, 4_099, 12_288], p=8, s=2, hier_k=k),
                        StepOptions(seed=7, lr=1e-2))
        for _ in range(steps // 100):
            step.run(100)
        eng.synchronize()
        S = step.sync_info()[0].shard_elems
        out += [eng.d2h(step.buffers()["master"], r, S) for r in range(8)]
        step.close()
        eng.close()
    eng = m.Engine(n_ranks=8, arena_bytes=128 << 20, devices=[0, 1])
    n = 8 * 4096
    a, b = eng.alloc(4 * n), eng.alloc(4 * n)
    for r in range(8):
        eng.generate(a, r, n, "f32", seed=11, step=r)
        eng.memset(b, r, 4 * n)
    ranks = list(range(8))
    rs = plan_reduce_scatter(eng, ranks, [eng.ptr(a, r) for r in ranks], n, [eng.ptr(b, r) for r in ranks], "f32",
                             mode=RS_ACCUMULATE, scale=-0.25)
    ag = plan_all_gather(eng, ranks, [eng.ptr(b, r) for r in ranks], 4 * n // 8, [eng.ptr(a, r) for r in ranks])
    for _ in range(chain):  # b -= RS(a) / 4 (~ -b); a = AG(b): every launch reads the previous one's output
        rs.run(1)
        ag.run(1)
    eng.synchronize()
    out += [eng.d2h(a, r, n) for r in ranks]
    rs.close()
    ag.close()
    eng.close()
    return out


def test_relaxed_barriers_match_fenced_under_stress(m, monkeypatch):
    relaxed = _run(m, monkeypatch, "0", 1000, 1000)
    fenced = _run(m, monkeypatch, "1", 1000, 1000)
    for x, y in zip(relaxed, fenced):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert all(np.isfinite(x).all() for x in relaxed)


def _tail_run(m, monkeypatch, variant, steps):
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_TAIL_OVERLAP", "0" if variant == "in_order" else "1")
    monkeypatch.setenv("MICS_TAIL_FUSED", "1" if variant == "k9" else "0")
    eng = m.Engine(n_ranks=8, arena_bytes=256 << 20, devices=[0, 1])
    # p=2: each position's 4 replicas span both GPUs; the 300k / 131k layers give several
    # K9 blocks per owner slice
    step = MicsStep(eng, Workload("tail stress", [300_000, 9_000, 131_072, 4_099], p=2, s=2),
                    StepOptions(seed=9, lr=1e-2))
    for _ in range(steps // 100):
        step.run(100)
    eng.synchronize()
    S = step.sync_info()[0].shard_elems
    b = step.buffers()
    out = [eng.d2h(b[k], r, S) for k in ("master", "exp_avg_sq") for r in range(8)]
    out += [eng.d2h(b["param_bf16"], r, S, "bf16") for r in (0, 5)]
    step.close()
    eng.close()
    return out


def test_k9_block_flags_match_under_stress(m, monkeypatch):
    """K9's relaxed per-block flags and item tickets (k_fbnd) over 500 back-to-back
    replayed steps on two GPUs of one process: the same bits as the two-kernel boundary
    and the in-order step.  A fold read before its owner's flag, or an Adam block before
    the fold, would compound into different bits."""
    ref = _tail_run(m, monkeypatch, "in_order", 500)
    for v in ("two_kernel", "k9"):
        got = _tail_run(m, monkeypatch, v, 500)
        for x, y in zip(ref, got):
            assert np.array_equal(x.view(np.uint16), y.view(np.uint16)), v
    assert all(np.isfinite(x.astype(np.float32)).all() for x in ref[:16])
