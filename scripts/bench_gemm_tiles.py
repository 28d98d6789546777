"""256- vs auto-chosen (128 where it quantises better) output tile widths on
the TP 3:1 rank-0 shapes and the 1-GPU shapes, sustained (power-capped).

    python scripts/bench_gemm_tiles.py
"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

CASES = [  # (tag, M, N, K, a_mn, b_mn)
    ("r0 o dgrad", 2048, 3072, 4096, 0, 0), ("r0 gu fwd", 2048, 16512, 4096, 0, 0),
    ("r0 qkv fwd", 2048, 9216, 4096, 0, 0), ("r0 down dgrad", 2048, 8256, 4096, 0, 0),
    ("r0 o fwd", 2048, 4096, 3072, 0, 1), ("r1 o dgrad", 2048, 1024, 4096, 0, 0),
    ("qkv fwd", 2048, 12288, 4096, 0, 0), ("gu fwd", 2048, 22016, 4096, 0, 0),
    ("o fwd", 2048, 4096, 4096, 0, 1),
]


def timed(fn, seconds=0.6):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < 0.2:
        fn()
        n += 1
    torch.cuda.synchronize()
    iters = max(5, int(n * seconds / 0.2))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for tag, M, N, K, amn, bmn in CASES:
    A = (torch.randn(K, M) if amn else torch.randn(M, K)).cuda().bfloat16()
    B = (torch.randn(K, N) if bmn else torch.randn(N, K)).cuda().bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    def go():
        assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), amn, M if amn else K, 0, 0,
                                B.data_ptr(), bmn, N if bmn else K, 0, 0, C.data_ptr(), N, 0, 0,
                                0, 0, 1.0, 0, None) == 0
    out = {"tag": tag, "M": M, "N": N, "K": K}
    for auto, mc in ((0, 1), (1, 1), (1, 2)):
        L.hexexec_k_gemm_tile_auto(auto)
        L.hexexec_k_gemm_multicast(mc)
        t = timed(go)
        out[f"tflops_auto{auto}_mc{mc}"] = round(2.0 * M * N * K / t / 1e9, 1)
    L.hexexec_k_gemm_multicast(1)
    print(json.dumps(out), flush=True)
L.hexexec_k_gemm_tile_auto(0)
