"""Time the tcgen05 GEMM on the step's shapes (CUDA events, L2 flushed).

    python scripts/bench_gemm.py            # prints one JSON line per case
"""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

PEAK = 1661.7


WS = None


def set_split(mode):
    """mode: -1 auto tail split (with workspace), 0 off"""
    global WS
    if WS is None:
        WS = (torch.zeros(148 * 128 * 256, device="cuda"),
              torch.zeros(148 * 8, device="cuda", dtype=torch.int32))
    assert L.hexexec_k_gemm_split(mode, WS[0].data_ptr(), WS[0].numel() * 4, WS[1].data_ptr(),
                                  WS[1].numel()) == 0


def run(M, N, K, a_mn=0, b_mn=0, c32=0, beta=0, iters=10, tag=""):
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).cuda().bfloat16()
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).cuda().bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if c32 else torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
    lda = M if a_mn else K
    ldb = N if b_mn else K

    def go():
        assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), a_mn, lda, 0, 0, B.data_ptr(), b_mn,
                                ldb, 0, 0, C.data_ptr(), N, 0, 0, c32, beta, 1.0, 0, None) == 0
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
    return {"tag": tag, "M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn, "c32": c32,
            "beta": beta, "ms": round(ms, 4), "tflops": round(tf, 1), "frac": round(tf / PEAK, 3)}


CASES = [
    ("qkv fwd", 2048, 12288, 4096, 0, 0, 0, 0),
    ("o fwd bf16", 2048, 4096, 4096, 0, 1, 0, 0),
    ("o wgrad beta", 4096, 4096, 2048, 1, 1, 1, 1),
    ("o wgrad nobeta", 4096, 4096, 2048, 1, 1, 1, 0),
    ("qkv wgrad beta", 12288, 4096, 2048, 1, 1, 1, 1),
    ("o fwd fp32", 2048, 4096, 4096, 0, 1, 1, 0),
    ("gu fwd", 2048, 22016, 4096, 0, 0, 0, 0),
    ("down fwd fp32", 2048, 4096, 11008, 0, 1, 1, 0),
    ("down dgrad", 2048, 11008, 4096, 0, 0, 0, 0),
    ("gu dgrad", 2048, 4096, 22016, 0, 1, 0, 0),
    ("down wgrad beta", 11008, 4096, 2048, 1, 1, 1, 1),
    ("gu wgrad beta", 22016, 4096, 2048, 1, 1, 1, 1),
    ("gu wgrad nobeta", 22016, 4096, 2048, 1, 1, 1, 0),
    ("gu wgrad bf16", 22016, 4096, 2048, 1, 1, 0, 0),
    ("lm head fp32", 2048, 32000, 4096, 0, 0, 1, 0),
    ("lm head bf16", 2048, 32000, 4096, 0, 0, 0, 0),
]

if __name__ == "__main__":
    sel = sys.argv[1:]
    for c in CASES:
        if not sel or any(s in c[0] for s in sel):
            row = {}
            for mode, name in ((0, "nosplit"), (-1, "split")):
                set_split(mode)
                r = run(*c[1:], tag=c[0])
                row[name] = r["tflops"]
            r.update(row)
            print(json.dumps(r), flush=True)
