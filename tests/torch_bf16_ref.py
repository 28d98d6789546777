"""TEST INFRASTRUCTURE — the bf16 floor: the same training step written in
plain PyTorch (autograd, torch.autocast bf16 on cuda, fp32 master weights
and fp32 gradient accumulation), from the oracle's initial weights and
tokens.  It measures how far a *standard* bf16 mixed-precision step lands
from the fp32 oracle (oracle/numeric.py) at a given shape, so the parity
tests can state the executor's error next to PyTorch's own bf16 error on the
same step.  Model math = oracle/numeric.py:
RMSNorm, rotate-half RoPE, causal MHA, SwiGLU over 64-column gate/up chunks,
vocab CE (mean over the global batch's tokens), on one device.
Not product code: only tests/ import it."""
from __future__ import annotations

import numpy as np


def step_grads(st, device="cuda", dtype="bf16"):
    """fwd + bwd of the global batch of oracle Step `st` in torch on one
    device; returns (global mean loss, {name: fp32 gradient of the global
    mean loss} = the oracle's DP-reduced gradient)."""
    import torch
    import torch.nn.functional as F
    m = st.m
    S, H, nh = m["seq_len"], m["hidden_dim"], m["num_heads"]
    d = H // nh
    eps = m["norm_eps"]
    # every pipeline's gradient is weighted by batch_i / global_batch, so the
    # reduced gradient is that of the global mean loss: one pass over the
    # global batch in micro-batches of pipeline 0's size gives the same math
    p = st.plan["pipelines"][0]
    B = st.plan["global_batch"]
    P = {k: torch.tensor(v, device=device, requires_grad=True) for k, v in st.W.items()}
    half = d // 2
    inv = st.m["rope_theta"] ** (-2.0 * np.arange(half, dtype=np.float64) / d)
    ang = np.arange(S, dtype=np.float64)[:, None] * inv[None]
    cos = torch.tensor(np.cos(ang), dtype=torch.float32, device=device)
    sin = torch.tensor(np.sin(ang), dtype=torch.float32, device=device)
    adt = torch.bfloat16 if dtype == "bf16" else torch.float32

    def rms(x, g):
        xf = x.float()
        r = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
        return (xf * r * g).to(adt)

    def rope(x):  # x [mb, nh, S, d]
        a, b = x[..., :half].float(), x[..., half:].float()
        return torch.cat([a * cos - b * sin, b * cos + a * sin], -1).to(adt)

    L = m["num_layers"]
    count = B * S
    toks = torch.tensor(st.tokens(0, 0, B), device=device, dtype=torch.long)
    total = 0.0
    mbs = p["micro_batch"] if B % p["micro_batch"] == 0 else 1
    for i in range(B // mbs):
        tok = toks[i * mbs:(i + 1) * mbs]
        inp, tgt = tok[:, :S].reshape(-1), tok[:, 1:].reshape(-1)
        x = P["embed"][inp]
        for l in range(L):
            pre = f"layers.{l}."
            xn = rms(x, P[pre + "attn_norm"][0])
            qkv = xn @ P[pre + "wqkv"].to(adt).T
            t = qkv.reshape(mbs, S, nh, 3, d).permute(0, 2, 3, 1, 4)
            q, k, v = rope(t[:, :, 0]), rope(t[:, :, 1]), t[:, :, 2]
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            attn = o.transpose(1, 2).reshape(mbs * S, nh * d)
            x = x + (attn @ P[pre + "wo"].to(adt)).float()
            hn = rms(x, P[pre + "mlp_norm"][0])
            gu = (hn @ P[pre + "wgu"].to(adt).T).reshape(-1, m["ffn_dim"] // 64, 2, 64)
            g, u = gu[:, :, 0].reshape(-1, m["ffn_dim"]), gu[:, :, 1].reshape(-1, m["ffn_dim"])
            a = (F.silu(g.float()) * u.float()).to(adt)
            x = x + (a @ P[pre + "wdown"].to(adt)).float()
        xf = rms(x, P["final_norm"][0])
        logits = (xf @ P["lm_head"].to(adt).T).float()
        loss = F.cross_entropy(logits, tgt, reduction="sum")
        (loss / count).backward()
        total += float(loss.detach())
    return total / count, {k: v.grad.detach().float().cpu().numpy() for k, v in P.items()}
