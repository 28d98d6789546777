"""Weight-gradient GEMMs: 8 micro-batches accumulated with 8 beta GEMMs
(K = 2048 each, fp32 TMA reduce-add into G) vs one GEMM over the
concatenated tokens (K = 16384, one fp32 store).  Sustained loop.

    python scripts/bench_wgrad_concat.py
"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402


def timed(fn, seconds=1.0):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < 0.3:
        fn()
        n += 1
    torch.cuda.synchronize()
    iters = max(3, int(n * seconds / 0.3))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for tag, Mw, N, K, G in [("gu wgrad", 22016, 4096, 2048, 8), ("o wgrad", 4096, 4096, 2048, 8),
                         ("down wgrad", 11008, 4096, 2048, 8), ("qkv wgrad", 12288, 4096, 2048, 8)]:
    A = torch.randn(G * K, Mw, device="cuda").bfloat16()   # dY tokens x out (MN-major A)
    B = torch.randn(G * K, N, device="cuda").bfloat16()    # X tokens x in (MN-major B)
    C = torch.zeros(Mw, N, device="cuda", dtype=torch.float32)

    def per_mb():
        for i in range(G):
            a = A[i * K:(i + 1) * K]
            b = B[i * K:(i + 1) * K]
            assert L.hexexec_k_gemm(Mw, N, K, 1, 1, a.data_ptr(), 1, Mw, 0, 0, b.data_ptr(), 1, N,
                                    0, 0, C.data_ptr(), N, 0, 0, 1, 1, 1.0, 0, None) == 0

    def concat():
        assert L.hexexec_k_gemm(Mw, N, G * K, 1, 1, A.data_ptr(), 1, Mw, 0, 0, B.data_ptr(), 1, N,
                                0, 0, C.data_ptr(), N, 0, 0, 1, 0, 1.0, 0, None) == 0
    f = 2.0 * Mw * N * K * G
    t1 = timed(per_mb)
    t2 = timed(concat)
    print(json.dumps({"tag": tag, "per_mb_ms": round(t1, 3), "concat_ms": round(t2, 3),
                      "per_mb_tflops": round(f / t1 / 1e9), "concat_tflops": round(f / t2 / 1e9)}),
          flush=True)
