"""GPU parity of the MiCS step with compute (csrc/step.cpp, cfg.compute): layer GEMMs
on the tcgen05 tensor cores (K7) produce the gradients that the 2-hop sync reduces.

The model: layer l is W_l = its gathered bf16 parameters viewed as [E_l / h, h];
every layer reads the micro-step input X [T, h]; loss 1/2 sum_l ||X W_lᵀ||^2, so
Y_l = X W_lᵀ (bf16), dX = sum_l Y_l W_l, dW_l = Y_lᵀ X.  The reference has no GEMM
(SURVEY §2b K7), so:
  * the GEMM outputs (Y, dX, dW) are checked against an fp32 restatement with a
    stated tolerance (fp32 accumulation order differs; Y may differ by one bf16 ulp);
  * the communication path is checked BIT-EXACTLY on the gradients the GEMMs
    actually produced: RS fold, micro-step accumulation, boundary fold and Adam are
    replayed on the CPU from the GPU's gradient slots and must match to the bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bf16_bits_to_f32(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(a):  # RNE, finite inputs
    b = np.ascontiguousarray(a, np.float32).view(np.uint32)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def reduce_and_adam(oracle, n, p, s, segs, grads, init, opts, step=1):
    """Bit-exact CPU replay of the 2-hop sync + Adam on given per-(t, rank) gradients."""
    S = sum(c for _, c, _, _ in segs)
    acc = np.zeros((n, S), np.float32)
    for r in range(n):
        j, g = r % p, r // p
        for t in range(s):
            fold = np.zeros(S, np.float32)
            for ln, c, so, go in segs:
                e = np.arange(c)
                valid = (j * c + e) < ln
                f = grads[t][g * p + 0][go + j * c + e].copy()
                for i in range(1, p):
                    f = f + grads[t][g * p + i][go + j * c + e]
                fold[so:so + c] = np.where(valid, f, np.float32(0))
            acc[r] = (np.float32(0) + fold) if t == 0 else (acc[r] + fold)
    out = []
    for r in range(n):
        j = r % p
        f = acc[j].copy()
        for q in range(1, n // p):
            f = f + acc[j + q * p]
        out.append(oracle.adam(init[r][0], init[r][1], init[r][2], f, opts.lr, opts.beta1, opts.beta2, opts.eps,
                               opts.weight_decay, step, 1.0 / (n * s), want_bf16=True))
    return out


def layer_weights(pbf16, segs, h, p, n_of):
    """W_l of partition group containing rank r: the concatenated bf16 shards."""
    Ws = []
    for ln, c, so, _ in segs:
        full = np.concatenate([pbf16[n_of(i)][so:so + c] for i in range(p)])[:ln]
        Ws.append(bf16_bits_to_f32(full).reshape(ln // h, h))
    return Ws


@pytest.mark.parametrize("recompute,grad_dtype,graph,ce,comm_sms", [
    (False, "f32", "1", "1", "16"), (True, "f32", "0", "1", "16"), (False, "bf16", "1", "1", "0"),
    (False, "f32", "1", "0", "0")])
def test_compute_step(oracle, monkeypatch, recompute, grad_dtype, graph, ce, comm_sms):
    """ce: flat gathers on the copy engines (default) or k_copy; comm_sms: SMs left to the
    overlapped reduce-scatters."""
    monkeypatch.setenv("MICS_CE_GATHER", ce)
    monkeypatch.setenv("MICS_COMM_SMS", comm_sms)
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    monkeypatch.setenv("MICS_GRAPH", graph)
    n, p, s, h = 8, 2, 2, 64
    layers = [h * 40, h * 37, h * 56]
    wl = Workload("cmp", layers, p=p, s=s, grad_dtype=grad_dtype, hidden=h, micro_batch=8, seq_len=16)
    T = wl.tokens
    opts = StepOptions(seed=91, lr=1e-3, compute=True, recompute=recompute)
    eng = Engine(n_ranks=n, device=0, arena_bytes=256 << 20)
    step = MicsStep(eng, wl, opts)
    info, segs = step.sync_info()
    S, G = info.shard_elems, info.grad_elems
    b = step.buffers()
    gdt = "bf16" if grad_dtype == "bf16" else "f32"
    for stepno in (1, 2):
        pb = [eng.d2h(b["param_bf16"], r, S, "bf16") for r in range(n)]
        init = [(eng.d2h(b["master"], r, S), eng.d2h(b["exp_avg"], r, S), eng.d2h(b["exp_avg_sq"], r, S))
                for r in range(n)]
        step.run(1)
        eng.synchronize()
        # the gradients the GEMMs produced: slot t holds micro-step t (s = 2 = slots)
        grads = np.zeros((s, n, G), np.float32)
        for t in range(s):
            for r in range(n):
                raw = eng.d2h(b["grads"], r, G, gdt, off=t * G * (2 if gdt == "bf16" else 4))
                grads[t, r] = bf16_bits_to_f32(raw) if gdt == "bf16" else raw
        # (1) GEMM outputs vs an fp32 restatement (tolerance)
        for r in range(n):
            g = r // p
            Ws = layer_weights(pb, segs, h, p, lambda i: g * p + i)
            for t in range(s):
                X = bf16_bits_to_f32(oracle.gen_bf16(91 ^ 0xA11CE, r, t, 254, 0, T * h)).reshape(T, h)
                for (ln, c, so, go), W in zip(segs, Ws):
                    Y = bf16_bits_to_f32(f32_to_bf16_bits(X @ W.T))
                    dW = (Y.T @ X).ravel()
                    bound = 2e-2 * (np.abs(Y).T @ np.abs(X)).ravel() + 1e-5
                    if gdt == "bf16":
                        bound += np.abs(dW) * 2.0 ** -8
                    got = grads[t, r, go:go + ln]
                    assert np.all(np.abs(got - dW) <= bound), (stepno, r, t, np.abs(got - dW).max())
                    assert not np.any(grads[t, r, go + ln:go + p * c]), "gradient padding must stay zero"
        # (2) communication path + Adam: bit-exact on the GPU's own gradients
        want = reduce_and_adam(oracle, n, p, s, segs, grads, init, opts, step=stepno)
        for r in range(n):
            wp, wm, wv, wb = want[r]
            assert np.array_equal(eng.d2h(b["master"], r, S).view(np.uint32), wp.view(np.uint32)), (stepno, r)
            assert np.array_equal(eng.d2h(b["exp_avg_sq"], r, S).view(np.uint32), wv.view(np.uint32)), (stepno, r)
            assert np.array_equal(eng.d2h(b["param_bf16"], r, S, "bf16"), wb), (stepno, r)
    st = step.stats()
    per_layer = sum(6 * T * e for e in layers) * (4 / 3 if recompute else 1)
    assert abs(st.compute_flops - n * s * per_layer) < 1e-6 * st.compute_flops
    assert st.gemm_launches == n * s * len(layers) * (4 if recompute else 3)
    # an eager host-input step after the graph was captured (fresh events), then a profile
    from paper_2205_00119_b200.engine import host_alloc, host_free
    host, hptr = host_alloc(T * h * 2)
    host[:] = oracle.gen_bf16(5, 0, 0, 254, 0, T * h).view(np.uint8)
    step.run_host(hptr, 1)
    eng.synchronize()
    host_free(hptr)
    prof = step.profile()
    assert prof["gemm_ms"] > 0 and prof["allgather_ms"] > 0 and prof["reducescatter_ms"] > 0
    step.close()
    eng.close()


def test_compute_step_rejects_bad_hidden():
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.errors import Error
    from paper_2205_00119_b200.step import MicsStep, StepOptions, Workload
    eng = Engine(n_ranks=8, device=0, arena_bytes=64 << 20)
    with pytest.raises(Error):
        MicsStep(eng, Workload("bad", [64 * 40 + 3], p=2, s=2, hidden=64, seq_len=16), StepOptions(compute=True))
    eng.close()
