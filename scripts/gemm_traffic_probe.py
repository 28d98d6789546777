"""The twelve TP linear GEMMs of one layer and micro-batch of the N=1 bench
step (llama7b_4l_1gpu: M = 2048 tokens, H 4096, F 11008), each launched once
after a warm-up round, in a fixed order, for an ncu --set full capture of their
DRAM traffic:

    ncu --set full --clock-control none -k regex:gemm_kernel -s 12 -c 12 \\
        -o gpurun_out/r02_gemm_probe python scripts/gemm_traffic_probe.py

Prints the shapes with their algorithmic bytes (A + B read once, C written
once; fp32 C accumulated with beta = read + write; a fp32 residual R read
once), which scripts/gemm_traffic_summary.py joins with the ncu report."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

T, H, F = 2048, 4096, 11008
# (tag, M, N, K, a_mn, b_mn, c_fp32, beta, residual)
SHAPES = [
    ("fwd qkv", T, 3 * H, H, 0, 0, 0, 0, 0),
    ("fwd o (+R)", T, H, H, 0, 1, 1, 0, 1),
    ("fwd gate-up", T, 2 * F, H, 0, 0, 0, 0, 0),
    ("fwd down (+R)", T, H, F, 0, 1, 1, 0, 1),
    ("dgrad down", T, F, H, 0, 0, 0, 0, 0),
    ("dgrad gate-up", T, H, 2 * F, 0, 1, 0, 0, 0),
    ("dgrad o", T, H, H, 0, 0, 0, 0, 0),
    ("dgrad qkv", T, H, 3 * H, 0, 1, 0, 0, 0),
    ("wgrad down", F, H, T, 1, 1, 1, 1, 0),
    ("wgrad gate-up", 2 * F, H, T, 1, 1, 1, 1, 0),
    ("wgrad o", H, H, T, 1, 1, 1, 1, 0),
    ("wgrad qkv", 3 * H, H, T, 1, 1, 1, 1, 0),
]


def algorithmic_bytes(M, N, K, c32, beta, res):
    c = M * N * (4 if c32 else 2)
    return 2 * M * K + 2 * N * K + c * (2 if beta else 1) + (M * N * 4 if res else 0)


def main():
    bufs = []
    for tag, M, N, K, amn, bmn, c32, beta, res in SHAPES:
        A = torch.randn(M * K, device="cuda").bfloat16()
        B = torch.randn(N * K, device="cuda").bfloat16()
        C = torch.zeros(M * N, device="cuda", dtype=torch.float32 if c32 else torch.bfloat16)
        bufs.append((A, B, C))
    out = []
    for rnd in range(2):  # round 0: warm-up, round 1: the captured launches
        for (tag, M, N, K, amn, bmn, c32, beta, res), (A, B, C) in zip(SHAPES, bufs):
            lda = M if amn else K
            ldb = N if bmn else K
            assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), amn, lda, 0, 0, B.data_ptr(), bmn,
                                    ldb, 0, 0, C.data_ptr(), N, 0, 0, c32, beta, 1.0, 0, None) == 0
            if rnd:
                # the kernel-level entry has no residual operand: the probe's
                # bytes leave R out (in the step these two also read R once)
                out.append({"tag": tag, "M": M, "N": N, "K": K, "flops": 2.0 * M * N * K,
                            "algorithmic_bytes": algorithmic_bytes(M, N, K, c32, beta, 0),
                            "in_step_algorithmic_bytes": algorithmic_bytes(M, N, K, c32, beta, res)})
    torch.cuda.synchronize()
    print(json.dumps({"shapes": out}))


if __name__ == "__main__":
    main()
