"""Time the HBM-bound kernels of one layer at the Llama-7B step shape
(M = 2048 tokens, H = 4096, F = 11008, V = 32000) through the C ABI and print
achieved GB/s of algorithmic traffic (bytes each kernel must move once)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main(M=2048, H=4096, F=11008, V=32000, nh=32, d=128, S=2048):
    p = lambda t: t.data_ptr()  # noqa: E731
    dev = "cuda"
    x = torch.randn(M, H, device=dev)
    y = torch.randn(M, H, device=dev).bfloat16()
    g = torch.rand(H, device=dev) + 0.5
    xo = torch.empty_like(x)
    out = torch.empty(M, H, device=dev, dtype=torch.bfloat16)
    rstd = torch.empty(M, device=dev)
    dy = torch.randn(M, H, device=dev).bfloat16()
    dres = torch.randn(M, H, device=dev)
    dx = torch.empty_like(x)
    dxb = torch.empty(M, H, device=dev, dtype=torch.bfloat16)
    dg = torch.zeros(H, device=dev)
    qkv = torch.randn(M, nh * 3 * d, device=dev).bfloat16()
    gu = torch.randn(M, 2 * F, device=dev).bfloat16()
    a = torch.empty(M, F, device=dev, dtype=torch.bfloat16)
    da = torch.randn(M, F, device=dev).bfloat16()
    dgu = torch.empty_like(gu)
    logits = torch.randn(M, V, device=dev)
    tok = torch.randint(0, V, (M // S, S + 1), device=dev, dtype=torch.int32)
    dl = torch.empty(M, V, device=dev, dtype=torch.bfloat16)
    loss = torch.zeros(1, device=dev)
    scr = torch.zeros(5 * M, device=dev)
    res = {}

    def rec(name, ms, nbytes):
        res[name] = {"us": round(ms * 1e3, 1), "GB/s": round(nbytes / ms / 1e6, 0)}

    rec("rmsnorm_fwd", timeit(lambda: L.hexexec_k_rmsnorm_fwd(
        p(x), p(y), p(xo), p(g), p(out), p(rstd), M, H, 1e-5, None)), M * H * (4 + 2 + 4 + 2))
    rec("rmsnorm_bwd", timeit(lambda: L.hexexec_k_rmsnorm_bwd(
        p(dy), None, p(x), p(rstd), p(g), p(dres), p(dx), p(dxb), p(dg), M, H, None)),
        M * H * (2 + 4 + 4 + 4 + 2))
    rec("rope", timeit(lambda: L.hexexec_k_rope(p(qkv), M, S, nh, d, 10000.0, 0, None)),
        M * nh * 2 * d * 2 * 2)
    rec("swiglu_fwd", timeit(lambda: L.hexexec_k_swiglu_fwd(p(gu), p(a), M, F, None)),
        M * F * 2 * 3)
    rec("swiglu_bwd", timeit(lambda: L.hexexec_k_swiglu_bwd(p(gu), p(da), p(dgu), M, F, None)),
        M * F * 2 * 5)
    rec("ce", timeit(lambda: L.hexexec_k_ce(p(logits), V, 0, p(tok), M, S, 1.0 / M, p(dl),
                                          p(loss), p(scr), None)), M * V * (4 + 4 + 2))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
