"""K7 GEMM throughput on the step's layer shapes vs torch.matmul (cuBLAS), bf16.

    python tools/gemm_bench.py            (one GPU)

Times back-to-back launches between CUDA events on the launching stream (inputs
re-used: the operands of these shapes stay L2-resident, as they do in the step).
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2205_00119_b200.engine import Engine
    from paper_2205_00119_b200.gemm import gemm_bf16
    eng = Engine(n_ranks=1, device=0, arena_bytes=64 << 20)
    ext = torch.cuda.ExternalStream(eng.stream())
    T, h = 4096, 1024
    cases = [  # name, M, N, K, a_mn, b_mn
        ("square 8192^3", 8192, 8192, 8192, False, False),
        ("fwd Y=X.W^T (BERT block)", T, 12301, h, False, False),
        ("dgrad dX=dY.W", T, h, 12301, False, True),
        ("wgrad dW=dY^T.X", 12301, h, T, True, True),
        ("GPT-2 1.5B dgrad (h=1600)", 8192, 1600, 19213, False, True),
        ("GPT-2 1.5B wgrad (h=1600)", 19213, 1600, 8192, True, True),
    ]
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    for name, M, N, K, a_mn, b_mn in cases:
        lda = (M if a_mn else K) + 7 & ~7
        ldb = (N if b_mn else K) + 7 & ~7
        ldc = N + 7 & ~7
        a = torch.randn((K if a_mn else M), lda, device="cuda").to(torch.bfloat16)
        b = torch.randn((K if b_mn else N), ldb, device="cuda").to(torch.bfloat16)
        c = torch.empty(M, ldc, device="cuda", dtype=torch.float32 if "wgrad" in name else torch.bfloat16)
        out = "f32" if c.dtype == torch.float32 else "bf16"
        torch.cuda.synchronize()

        def ours(n):
            for _ in range(n):
                gemm_bf16(eng, a.data_ptr(), lda, a_mn, b.data_ptr(), ldb, b_mn, c.data_ptr(), ldc, out, M, N, K)
        A = a[:, :M].t() if a_mn else a[:, :K]
        B = b[:, :N] if b_mn else b[:, :K].t()

        def cublas(n):
            with torch.cuda.stream(ext):
                for _ in range(n):
                    torch.matmul(A, B)
        res = {}
        for nm, fn in (("k7", ours), ("cublas", cublas)):
            fn(3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record(ext)
            fn(reps)
            e1.record(ext)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res[nm] = {"ms": ms, "tflops": 2.0 * M * N * K / ms / 1e9}
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn, "out": out,
                          "k7_ms": res["k7"]["ms"], "k7_tflops": res["k7"]["tflops"],
                          "cublas_tflops": res["cublas"]["tflops"],
                          "frac_of_measured_peak": res["k7"]["tflops"] / pk["bf16_tflops"]}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
