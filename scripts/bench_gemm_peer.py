"""Cost of the TP peer copy in the GEMM epilogue (tp_reduce = "peer"): the
row-parallel / dgrad GEMMs of the 7B TP 3:1 plan with C stored locally only
vs also TMA-stored into a buffer on GPU 1 (peer access over NVLink).

    python scripts/bench_gemm_peer.py     # needs 2 GPUs; one JSON line per case
"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

CASES = [  # (tag, M, N, K, b_mn) -- rank 0 (3/4) and rank 1 (1/4) shards
    ("o_proj r0", 2048, 4096, 3072, 1), ("down r0", 2048, 4096, 8256, 1),
    ("qkv dgrad r0", 2048, 4096, 9216, 1), ("gu dgrad r0", 2048, 4096, 16512, 1),
    ("lm dgrad r0", 2048, 4096, 24000, 1), ("o_proj r1", 2048, 4096, 1024, 1),
]


def main():
    assert torch.cuda.device_count() >= 2
    rt = ctypes.CDLL("libcudart.so.12") if False else None  # noqa: F841
    torch.cuda.set_device(0)
    assert torch.cuda.can_device_access_peer(0, 1)
    # enable P2P: a cross-device copy makes torch enable peer access
    x1 = torch.zeros(16, device="cuda:1")
    x1.copy_(torch.ones(16, device="cuda:0"))
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda:0")
    for tag, M, N, K, bmn in CASES:
        A = torch.randn(M, K, device="cuda:0").bfloat16()
        B = torch.randn(K, N, device="cuda:0").bfloat16() if bmn else torch.randn(N, K, device="cuda:0").bfloat16()
        C = torch.zeros(M, N, device="cuda:0", dtype=torch.bfloat16)
        P = torch.zeros(M, N, device="cuda:1", dtype=torch.bfloat16)
        out = {"tag": tag, "M": M, "N": N, "K": K}
        for npeer in (0, 1):
            arr = (ctypes.c_void_p * 1)(P.data_ptr())
            assert L.hexexec_k_gemm_peers(arr, npeer) == 0

            def go():
                assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), 0, K, 0, 0, B.data_ptr(), bmn,
                                        N if bmn else K, 0, 0, C.data_ptr(), N, 0, 0, 0, 0, 1.0, 0,
                                        None) == 0
            for _ in range(3):
                go()
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                go()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e))
            ts.sort()
            out[f"ms_peer{npeer}"] = round(ts[len(ts) // 2], 4)
            out[f"tflops_peer{npeer}"] = round(2.0 * M * N * K / ts[len(ts) // 2] / 1e9, 1)
        torch.cuda.synchronize()
        out["peer_equal_local"] = bool(torch.equal(C.cpu(), P.cpu()))
        assert L.hexexec_k_gemm_peers(None, 0) == 0
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
