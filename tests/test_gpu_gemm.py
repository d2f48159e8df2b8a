"""K7 tcgen05 GEMM (csrc/gemm.cu) against a plain fp32 matmul of the same bf16
operands (the reference has no GEMM).

Tolerance: fp32 accumulation in a different order than torch's, so
|got - want| <= 1e-4 * (|A| |B|)[m, n] + 1e-6 for an f32 output; one bf16 rounding
(2^-8 relative) on top of that for a bf16 output.
"""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eng():
    from paper_2205_00119_b200.engine import Engine
    e = Engine(n_ranks=1, device=0, arena_bytes=64 << 20)
    yield e
    e.close()


def operand(rows, cols, ld, gen):
    """bf16 [rows, ld] storage holding a [rows, cols] matrix (padding = garbage)."""
    full = torch.randn(rows, ld, generator=gen, device="cuda").to(torch.bfloat16)
    return full, full[:, :cols]


def ld(cols, pad):
    return (cols + pad + 7) // 8 * 8  # TMA: 16-byte row strides


def run(eng, M, N, K, a_mn, b_mn, out, accumulate=False, pad=8, seed=0):
    from paper_2205_00119_b200.gemm import gemm_bf16
    g = torch.Generator(device="cuda").manual_seed(seed)
    # logical A [M, K]: K-major storage [M, lda>=K]; M-major storage [K, lda>=M]
    if a_mn:
        a_st, a_v = operand(K, M, ld(M, pad), g)
        A = a_v.t()
    else:
        a_st, A = operand(M, K, ld(K, pad), g)
    # logical B [K, N]: K-major storage [N, ldb>=K]; N-major storage [K, ldb>=N]
    if b_mn:
        b_st, B = operand(K, N, ld(N, pad), g)
    else:
        b_st, b_v = operand(N, K, ld(K, pad), g)
        B = b_v.t()
    ldc = N + pad
    cdt = torch.float32 if out == "f32" else torch.bfloat16
    C = torch.randn(M, ldc, generator=g, device="cuda").to(cdt)
    C0 = C.clone()
    torch.cuda.synchronize()
    gemm_bf16(eng, a_st.data_ptr(), a_st.stride(0), a_mn, b_st.data_ptr(), b_st.stride(0), b_mn, C.data_ptr(), ldc,
              out, M, N, K, accumulate)
    eng.synchronize()
    want = A.float() @ B.float()
    if accumulate:
        want = want + C0[:, :N].float()
    bound = (A.float().abs() @ B.float().abs()) * 1e-4 + 1e-6
    if accumulate:
        bound = bound + C0[:, :N].float().abs() * 1e-6
    got = C[:, :N].float()
    if out == "bf16":
        bound = bound + want.abs() * 2.0 ** -8
    err = (got - want).abs()
    assert bool((err <= bound).all()), f"max err {err.max().item()} (bound {bound[err > bound].min().item()})"
    assert torch.equal(C[:, N:], C0[:, N:]), "wrote outside [M, N]"


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
def test_gemm_layouts_tile_multiples(eng, a_mn, b_mn):
    run(eng, 256, 512, 192, a_mn, b_mn, "f32")


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_gemm_ragged_edges(eng, a_mn, b_mn, out):
    run(eng, 200, 300, 136, a_mn, b_mn, out, seed=1)


def test_gemm_accumulate(eng):
    run(eng, 384, 520, 256, False, True, "f32", accumulate=True, seed=2)


def test_gemm_many_tiles_persistent(eng):
    # more tiles than SMs (persistent loop, both accumulator buffers, ring wrap-around)
    run(eng, 2048, 4104, 320, False, False, "bf16", seed=3)


def test_gemm_rejects_bad_args(eng):
    from paper_2205_00119_b200.errors import Error
    from paper_2205_00119_b200.gemm import gemm_bf16
    x = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(Error):
        gemm_bf16(eng, x.data_ptr(), 64, False, x.data_ptr(), 64, False, x.data_ptr(), 64, "bf16", 64, 64, 64, True)
    with pytest.raises(Error):
        gemm_bf16(eng, x.data_ptr() + 2, 64, False, x.data_ptr(), 64, False, x.data_ptr(), 64, "bf16", 64, 64, 64)


def test_gemm_hidden_1600_accumulate(eng):
    """N = 1600 (GPT-2 1.5B hidden: 6.25 tiles of 256, a ragged last column of tiles); accumulate."""
    run(eng, 512, 1600, 320, False, True, "f32", accumulate=True, seed=6)
