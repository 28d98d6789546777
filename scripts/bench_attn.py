"""Time the fused causal attention kernels at the Llama-7B shard shape."""
import json
import math
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2409_01143_b200 import _lib as L  # noqa: E402


def main(mb=1, S=2048, nh=32, d=128, iters=10, variant=3, fwd_variant=3):
    L.hexexec_k_attn_variant(fwd_variant, variant)
    torch.manual_seed(0)
    qkv = torch.randn(mb * S, nh * 3 * d, device="cuda").bfloat16()
    out = torch.zeros(mb * S, nh * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(mb * nh, S, device="cuda")
    dout = torch.randn(mb * S, nh * d, device="cuda").bfloat16()
    delta = torch.zeros(mb * nh, S, device="cuda")
    dq = torch.zeros(mb * S, nh * d, device="cuda")
    dqkv = torch.zeros_like(qkv)
    sc = 1.0 / math.sqrt(d)

    def fwd():
        assert L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb,
                                    sc, None) == 0

    def bwd():
        assert L.hexexec_k_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(),
                                    lse.data_ptr(), delta.data_ptr(), dq.data_ptr(),
                                    dqkv.data_ptr(), S, nh, d, mb, sc, None) == 0
    res = {}
    flops = 2.0 * 2 * mb * nh * S * S * d / 2  # causal fwd: QK^T + PV, lower triangle
    for name, fn, f in (("fwd", fwd, flops), ("bwd", bwd, 2.5 * flops)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        res[name] = {"ms": round(ms, 4), "tflops": round(f / ms / 1e9, 1)}
    # library baseline on the same shape: flash-attn 2.8 (FA2 kernels, mma.sync
    # recompiled for sm_100), bf16, causal, fwd and bwd timed separately
    try:
        from flash_attn import flash_attn_func
        q, k, v = (torch.randn(mb, S, nh, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
                   for _ in range(3))
        go = torch.randn(mb, S, nh, d, device="cuda", dtype=torch.bfloat16)
        o = flash_attn_func(q, k, v, causal=True)
        o.backward(go)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            o = flash_attn_func(q, k, v, causal=True)
        e.record()
        torch.cuda.synchronize()
        tf = s.elapsed_time(e) / iters
        outs = [flash_attn_func(q, k, v, causal=True) for _ in range(iters)]
        torch.cuda.synchronize()
        s.record()
        for o in outs:
            o.backward(go)
        e.record()
        torch.cuda.synchronize()
        tb = s.elapsed_time(e) / iters
        res["flash_attn2"] = {"fwd_ms": round(tf, 4), "fwd_tflops": round(flops / tf / 1e9, 1),
                              "bwd_ms": round(tb, 4), "bwd_tflops": round(2.5 * flops / tb / 1e9, 1)}
    except Exception as ex:  # noqa: BLE001
        res["flash_attn2"] = {"error": str(ex)[:200]}
    print(json.dumps({"shape": [mb, S, nh, d], "fwd_variant": fwd_variant, "bwd_variant": variant,
                      **res}))


if __name__ == "__main__":
    # arguments: [fwd:]bwd variant pairs, e.g. 3:3 2:3 2:1
    for a in (sys.argv[1:] or ["3", "2", "1"]):
        f, _, b = a.rpartition(":")
        main(variant=int(b), fwd_variant=int(f) if f else 3)
