"""Small launches of the hand-written kernels for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python scripts/sanitize_kernels.py
    compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py attn

attention forward (v3, v2) and backward (v3, v2, v1) at S 256 (two key tiles,
diagonal masking), d 64 / 128; GEMMs with K / N tails; then one tiny training
step through the executor (all kernels of the step)."""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_01143_b200 import _lib as L  # noqa: E402


def attention():
    for d in (64, 128):
        mb, S, nh = 1, 256, 2
        qkv = torch.randn(mb * S, nh * 3 * d, device="cuda").bfloat16()
        out = torch.zeros(mb * S, nh * d, device="cuda", dtype=torch.bfloat16)
        lse = torch.zeros(mb * nh, S, device="cuda")
        dout = torch.randn(mb * S, nh * d, device="cuda").bfloat16()
        delta = torch.zeros(mb * nh, S, device="cuda")
        dq = torch.zeros(mb * S, nh * d, device="cuda")
        dqkv = torch.zeros_like(qkv)
        for fv, bv in ((3, 3), (2, 2), (2, 1)):
            assert L.hexexec_k_attn_variant(fv, bv) == 0
            assert L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb,
                                        1 / math.sqrt(d), None) == 0
            assert L.hexexec_k_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(),
                                        lse.data_ptr(), delta.data_ptr(), dq.data_ptr(),
                                        dqkv.data_ptr(), S, nh, d, mb, 1 / math.sqrt(d), None) == 0
            torch.cuda.synchronize()
    L.hexexec_k_attn_variant(3, 3)


def gemm():
    for M, N, K in ((256, 384, 192), (512, 256, 2752 // 8)):
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(N, K, device="cuda").bfloat16()
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        assert L.hexexec_k_gemm(M, N, K, 1, 1, A.data_ptr(), 0, K, 0, 0, B.data_ptr(), 0, K, 0, 0,
                                C.data_ptr(), N, 0, 0, 0, 0, 1.0, 0, None) == 0
        torch.cuda.synchronize()


def step():
    from paper_2409_01143_b200 import Executor
    cfg = os.path.join(ROOT, "configs")
    c = open(os.path.join(cfg, "clusters", "b200_1.json")).read()
    m = open(os.path.join(cfg, "models", "tiny.json")).read()
    p = open(os.path.join(cfg, "plans", "tiny_1.json")).read()
    ex = Executor(c, m, p, {"cuda_graph": False}, rank=0, world_size=1, device=0)
    loss = ex.step(ex.synth_tokens(0))
    ex.close()
    return loss


if __name__ == "__main__":
    what = sys.argv[1:] or ["attn", "gemm", "step"]
    out = {}
    if "attn" in what:
        attention()
        out["attention"] = "ok"
    if "gemm" in what:
        gemm()
        out["gemm"] = "ok"
    if "step" in what:
        out["step_loss"] = step()
    print(json.dumps(out))
