"""Sustained (power-capped) throughput of the tcgen05 GEMM vs cuBLAS
(torch.matmul, the library baseline) on the step's GEMM shapes: each case runs
back to back for ~1 s (no L2 flush: inside the step consecutive GEMMs do not
flush either), CUDA events around the whole loop, clocks as they settle.

    python scripts/bench_gemm_vs_cublas.py      # one JSON line per case
"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

# (tag, M, N, K, a_mn, b_mn)  -- C = A[M,K] B[N,K]^T, bf16 out
CASES = [
    ("qkv fwd", 2048, 12288, 4096, 0, 0),
    ("o fwd", 2048, 4096, 4096, 0, 1),
    ("gu fwd", 2048, 22016, 4096, 0, 0),
    ("down fwd", 2048, 4096, 11008, 0, 1),
    ("down dgrad", 2048, 11008, 4096, 0, 0),
    ("gu dgrad", 2048, 4096, 22016, 0, 1),
    ("o wgrad", 4096, 4096, 2048, 1, 1),
    ("gu wgrad", 22016, 4096, 2048, 1, 1),
    ("lm head", 2048, 32000, 4096, 0, 0),
    ("square 8192", 8192, 8192, 8192, 0, 0),
]


def timed(fn, seconds=1.0):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < 0.3:  # warm up into the power-capped regime
        fn()
        n += 1
    torch.cuda.synchronize()
    iters = max(5, int(n * seconds / 0.3))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    for tag, M, N, K, amn, bmn in CASES:
        A = (torch.randn(K, M) if amn else torch.randn(M, K)).cuda().bfloat16()
        B = (torch.randn(K, N) if bmn else torch.randn(N, K)).cuda().bfloat16()
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        lda = M if amn else K
        ldb = N if bmn else K

        def ours():
            assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), amn, lda, 0, 0, B.data_ptr(), bmn,
                                    ldb, 0, 0, C.data_ptr(), N, 0, 0, 0, 0, 1.0, 0, None) == 0
        a_ = A.t() if amn else A          # logical [M, K]
        bt = B if bmn else B.t()          # logical [K, N]

        def cublas():
            torch.matmul(a_, bt, out=C)
        f = 2.0 * M * N * K
        assert L.hexexec_k_gemm_raster(0) == 0
        t_n = timed(ours)
        assert L.hexexec_k_gemm_raster(8) == 0
        t_o = timed(ours)
        assert L.hexexec_k_gemm_multicast(2) == 0
        t_m = timed(ours)
        assert L.hexexec_k_gemm_multicast(1) == 0
        t_c = timed(cublas)
        print(json.dumps({"tag": tag, "M": M, "N": N, "K": K, "ours_us": round(t_o * 1e3, 1),
                          "cublas_us": round(t_c * 1e3, 1),
                          "ours_tflops": round(f / t_o / 1e9, 1),
                          "ours_nfastest_tflops": round(f / t_n / 1e9, 1),
                          "ours_amulticast_tflops": round(f / t_m / 1e9, 1),
                          "cublas_tflops": round(f / t_c / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
