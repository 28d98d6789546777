"""Time the tcgen05 GEMM on the step's TP shapes (CUDA events, L2 flushed)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

PEAK = 1661.7


def run(M, N, K, a_mn=0, b_mn=0, iters=20):
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).cuda().bfloat16()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).cuda().bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
    lda = M if a_mn else K
    ldb = N if b_mn else K

    def go():
        assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), a_mn, lda, 0, 0, B.data_ptr(), b_mn,
                                ldb, 0, 0, C.data_ptr(), N, 0, 0, 0, 0, 1.0, 0, None) == 0
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        go()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    ms = ts[len(ts) // 2]
    tf = 2.0 * M * N * K / ms / 1e9
    ref = torch.matmul(A.float().T if a_mn else A.float(), (B.float() if b_mn else B.float().T))
    err = ((C.float() - ref).abs().max() / ref.abs().max()).item()
    return {"M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn, "ms": round(ms, 4),
            "tflops": round(tf, 1), "frac": round(tf / PEAK, 3), "err": err}


if __name__ == "__main__":
    shapes = [(2048, 9216, 4096, 0, 0), (2048, 4096, 3072, 0, 1), (2048, 16512, 4096, 0, 0),
              (2048, 4096, 8256, 0, 1), (9216, 4096, 2048, 1, 1), (8192, 8192, 8192, 0, 0),
              (2048, 3072, 4096, 0, 0), (4096, 4096, 4096, 0, 0)]
    for s in shapes:
        print(json.dumps(run(*s)))
