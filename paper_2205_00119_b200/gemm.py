"""K7: the tcgen05 bf16 GEMM (csrc/gemm.cu) used by the step with compute.

C[m, n] (+)= sum_k A(m, k) B(k, n) on the engine's stream, device pointers,
row-major storage; either operand K-major or MN-major (include/mics.h,
mics_gemm_bf16).  The reference has no GEMM: this is checked
against an fp32 matmul, not against the reference.
"""
from __future__ import annotations

from ._lib import check, lib
from .engine import DTYPE, Engine


def gemm_bf16(engine: Engine, a: int, lda: int, a_mn: bool, b: int, ldb: int, b_mn: bool, c: int, ldc: int,
              c_dtype: str, m: int, n: int, k: int, accumulate: bool = False) -> None:
    """A(m,k) = a[m*lda+k] (K-major) or a[k*lda+m] (a_mn); B(k,n) = b[n*ldb+k] (K-major)
    or b[k*ldb+n] (b_mn); C(m,n) = c[m*ldc+n] in f32 or bf16."""
    check(lib.mics_gemm_bf16(engine.ctx, a, lda, int(a_mn), b, ldb, int(b_mn), c, ldc, DTYPE[c_dtype], m, n, k,
                             int(accumulate)))
