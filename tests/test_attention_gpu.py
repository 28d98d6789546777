"""Fused causal attention kernels (tcgen05) vs a plain PyTorch fp32 reference
on the same bf16 inputs.  Tolerance: outputs / gradients normwise rel 1e-2
(bf16 P and outputs), LSE abs 1e-3 (fp32 statistics)."""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _L():
    from paper_2409_01143_b200 import _lib
    return _lib


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def _ref(qkv, mb, S, nh, d, scale):
    t = qkv.float().view(mb, S, nh, 3, d)
    q, k, v = (t[:, :, :, i].transpose(1, 2) for i in range(3))  # [mb, nh, S, d]
    s = (q @ k.transpose(-1, -2)) * scale
    mask = torch.triu(torch.ones(S, S, device=qkv.device, dtype=torch.bool), 1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.transpose(1, 2).reshape(mb * S, nh * d), lse.reshape(mb * nh, S), (q, k, v)


@pytest.mark.parametrize("variant", [3, 2])
@pytest.mark.parametrize("mb,S,nh,d", [(1, 256, 2, 128), (2, 384, 3, 64), (1, 2048, 2, 128),
                                       (1, 2048, 32, 128), (1, 128, 1, 64)])
def test_attention_forward(cuda, mb, S, nh, d, variant):
    """v3 (P in TMEM, V double-buffered) and v2 forward kernels."""
    L = _L()
    assert L.hexexec_k_attn_variant(variant, 0) == 0
    torch.manual_seed(0)
    qkv = torch.randn(mb * S, nh * 3 * d, device=cuda).bfloat16()
    out = torch.zeros(mb * S, nh * d, device=cuda, dtype=torch.bfloat16)
    lse = torch.zeros(mb * nh, S, device=cuda)
    scale = 1.0 / math.sqrt(d)
    assert L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb,
                                scale, None) == 0
    torch.cuda.synchronize()
    L.hexexec_k_attn_variant(3, 0)
    ro, rl, _ = _ref(qkv, mb, S, nh, d, scale)
    assert _rel(out, ro) < 1e-2
    assert (lse / math.log2(math.e) - rl).abs().max().item() < 1e-3


@pytest.mark.parametrize("variant", [3, 2, 1])
@pytest.mark.parametrize("mb,S,nh,d", [(1, 256, 2, 128), (2, 384, 3, 64), (1, 2048, 2, 128),
                                       (1, 2048, 32, 128), (1, 128, 1, 64)])
def test_attention_backward(cuda, mb, S, nh, d, variant):
    """v3 (P^T in TMEM), v2 (dQ epilogue warpgroup) and v1 backward kernels."""
    L = _L()
    assert L.hexexec_k_attn_variant(0, variant) == 0
    torch.manual_seed(1)
    qkv = torch.randn(mb * S, nh * 3 * d, device=cuda).bfloat16()
    out = torch.zeros(mb * S, nh * d, device=cuda, dtype=torch.bfloat16)
    lse = torch.zeros(mb * nh, S, device=cuda)
    scale = 1.0 / math.sqrt(d)
    assert L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb,
                                scale, None) == 0
    dout = torch.randn(mb * S, nh * d, device=cuda).bfloat16()
    delta = torch.zeros(mb * nh, S, device=cuda)
    dq_acc = torch.zeros(mb * S, nh * d, device=cuda)
    dqkv = torch.zeros_like(qkv)
    assert L.hexexec_k_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                delta.data_ptr(), dq_acc.data_ptr(), dqkv.data_ptr(), S, nh, d,
                                mb, scale, None) == 0
    torch.cuda.synchronize()
    x = qkv.float().clone().requires_grad_(True)
    ro, _, _ = _ref(x, mb, S, nh, d, scale)
    ro.backward(dout.float())
    g = dqkv.float().view(mb * S, nh, 3, d)
    r = x.grad.view(mb * S, nh, 3, d)
    L.hexexec_k_attn_variant(0, 3)
    for part in range(3):
        assert _rel(g[:, :, part], r[:, :, part]) < 2e-2, part


def test_attention_forward_v3_matches_v2_bitwise(cuda):
    """P kept in TMEM (v3) vs P through shared memory (v2): the same bf16 P,
    the same MMAs, so the same output and LSE bit for bit (also a check that
    the next S product never overwrites P before O += P V has read it)."""
    L = _L()
    torch.manual_seed(3)
    mb, S, nh, d = 2, 2048, 8, 128
    qkv = torch.randn(mb * S, nh * 3 * d, device=cuda).bfloat16()
    outs = []
    for v in (2, 3, 3, 3):
        out = torch.zeros(mb * S, nh * d, device=cuda, dtype=torch.bfloat16)
        lse = torch.zeros(mb * nh, S, device=cuda)
        assert L.hexexec_k_attn_variant(v, 0) == 0
        assert L.hexexec_k_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), S, nh, d, mb,
                                    1.0 / math.sqrt(d), None) == 0
        torch.cuda.synchronize()
        outs.append((out, lse))
    L.hexexec_k_attn_variant(3, 0)
    for o, l in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(l, outs[0][1])
