"""Does a weight-gradient GEMM on a side stream overlap the attention
backward (a low-power, latency-bound kernel) on a power-capped B200?
Sequential vs concurrent (GEMM grid capped to `sms` SMs), back to back for ~1 s.

    python scripts/bench_overlap.py
"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402

S, nh, d, mb = 2048, 32, 128, 1
M = mb * S
qkv = (torch.randn(M, nh * 3 * d, device="cuda") * 0.5).bfloat16()
out = torch.randn(M, nh * d, device="cuda").bfloat16()
dout = torch.randn(M, nh * d, device="cuda").bfloat16()
lse = torch.zeros(mb * nh * S, device="cuda")
delta = torch.zeros(mb * nh * S, device="cuda")
dq = torch.zeros(M, nh * d, device="cuda")
dqkv = torch.zeros(M, nh * 3 * d, device="cuda").bfloat16()
assert L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb,
                            d ** -0.5, None) == 0
# wgrad shapes of one layer (gu: 22016 x 4096, K = 2048 tokens)
Mw, Nw, Kw = 22016, 4096, 2048
A = torch.randn(Kw, Mw, device="cuda").bfloat16()
B = torch.randn(Kw, Nw, device="cuda").bfloat16()
G = torch.zeros(Mw, Nw, device="cuda")
s_main = torch.cuda.Stream()
s_side = torch.cuda.Stream()


def attn(stream):
    assert L.hexexec_k_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                delta.data_ptr(), dq.data_ptr(), dqkv.data_ptr(), S, nh, d, mb,
                                d ** -0.5, stream.cuda_stream) == 0


def wgrad(stream, sms):
    L.hexexec_k_gemm_sm_limit(sms)
    assert L.hexexec_k_gemm(Mw, Nw, Kw, 1, 1, A.data_ptr(), 1, Mw, 0, 0, B.data_ptr(), 1, Nw, 0, 0,
                            G.data_ptr(), Nw, 0, 0, 1, 1, 1.0, 0, stream.cuda_stream) == 0
    L.hexexec_k_gemm_sm_limit(0)


def run(mode, sms, iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        if mode == "seq":
            attn(s_main)
            wgrad(s_main, 0)
        else:
            ev = torch.cuda.Event()
            ev.record(s_main)
            s_side.wait_event(ev)
            wgrad(s_side, sms)
            attn(s_main)
            ev2 = torch.cuda.Event()
            ev2.record(s_side)
            s_main.wait_event(ev2)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / iters * 1e3


for mode, sms in [("seq", 0), ("conc", 148), ("conc", 96), ("conc", 64), ("conc", 32), ("seq", 0)]:
    run(mode, sms, 20)
    ms = run(mode, sms, 300)
    print(json.dumps({"mode": mode, "gemm_sms": sms, "ms_per_pair": round(ms, 4)}), flush=True)
t = run("seq", 0, 5)
for name, fn in (("attn only", lambda: attn(s_main)), ("wgrad only", lambda: wgrad(s_main, 0))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(300):
        fn()
    torch.cuda.synchronize()
    print(json.dumps({"mode": name, "ms": round((time.perf_counter() - t0) / 300 * 1e3, 4)}))
