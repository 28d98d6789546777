"""Generate golden vectors for the tiny config with PyTorch fp32 autograd.

An independent restatement of the model (torch autograd, not the numpy
oracle's hand-written backward) on the same weights / tokens (oracle.rng).
Stores, per tensor, the gradient and updated weight at 512 fixed sampled
positions plus sum / sum-of-squares checksums, and the loss.  These pin the
numpy oracle (tests/test_oracle_numeric.py) and, transitively, the GPU path.

    python tests/golden/make_golden.py      # writes tests/golden/tiny_step.npz
"""
import json
import math
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bookkeeping as bk  # noqa: E402
from oracle import numeric as O  # noqa: E402
from oracle import rng  # noqa: E402

torch.set_default_dtype(torch.float32)


def rope(x, S, d, theta, pos):
    half = d // 2
    inv = theta ** (-2.0 * torch.arange(half, dtype=torch.float64) / d)
    ang = pos[:, None].double() * inv[None]
    c, s = torch.cos(ang).float(), torch.sin(ang).float()
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * c - b * s, b * c + a * s], -1)


def model_loss(W, tok, m):
    S, H, nh, L = m["seq_len"], m["hidden_dim"], m["num_heads"], m["num_layers"]
    d, F, eps = H // nh, m["ffn_dim"], m["norm_eps"]
    B = tok.shape[0]
    inp = torch.as_tensor(tok[:, :S].astype(np.int64))
    tgt = torch.as_tensor(tok[:, 1:].astype(np.int64)).reshape(-1)

    def norm(x, g):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g

    x = W["embed"][inp]                                     # [B, S, H]
    pos = torch.arange(S)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool), 1)
    for l in range(L):
        p = f"layers.{l}."
        xn = norm(x, W[p + "attn_norm"][0])
        qkv = (xn @ W[p + "wqkv"].T).view(B, S, nh, 3, d)
        q = rope(qkv[:, :, :, 0].transpose(1, 2), S, d, m["rope_theta"], pos)
        k = rope(qkv[:, :, :, 1].transpose(1, 2), S, d, m["rope_theta"], pos)
        v = qkv[:, :, :, 2].transpose(1, 2)
        s = (q @ k.transpose(-1, -2)) / math.sqrt(d)
        P = torch.softmax(s.masked_fill(mask, float("-inf")), -1)
        attn = (P @ v).transpose(1, 2).reshape(B, S, H)
        x = x + attn @ W[p + "wo"]
        hn = norm(x, W[p + "mlp_norm"][0])
        gu = (hn @ W[p + "wgu"].T).view(B, S, F // 64, 2, 64)
        g = gu[..., 0, :].reshape(B, S, F)
        u = gu[..., 1, :].reshape(B, S, F)
        x = x + (torch.nn.functional.silu(g) * u) @ W[p + "wdown"]
    xf = norm(x, W["final_norm"][0])
    logits = xf @ W["lm_head"].T
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), tgt)


def main():
    cfg = os.path.join(ROOT, "configs")
    m = bk.model_defaults(json.load(open(os.path.join(cfg, "models", "tiny.json"))))
    seed, step, B = 0, 0, 8
    W0 = O.init_weights(m, seed)
    W = {k: torch.tensor(v, requires_grad=True) for k, v in W0.items()}
    tok = rng.tokens(seed, step, 0, B, m["seq_len"], m["vocab_size"])
    loss = model_loss(W, tok, m)
    loss.backward()
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.95, 1e-8, 0.1
    out = {"loss": np.float64(loss.item())}
    g = np.random.default_rng(1234)
    for k, t in W.items():
        grad = t.grad.numpy().astype(np.float32)
        kind = k.split(".")[-1]
        w = 0.0 if kind in ("attn_norm", "mlp_norm", "final_norm") else wd
        mo = (1 - b1) * grad
        ve = (1 - b2) * grad * grad
        upd = (mo / (1 - b1)) / (np.sqrt(ve / (1 - b2)) + eps)
        neww = (W0[k] - lr * (upd + w * W0[k])).astype(np.float32)
        idx = g.choice(grad.size, size=min(512, grad.size), replace=False)
        out[f"{k}|idx"] = idx
        out[f"{k}|grad"] = grad.reshape(-1)[idx]
        out[f"{k}|w"] = neww.reshape(-1)[idx]
        out[f"{k}|gsum"] = np.float64(grad.astype(np.float64).sum())
        out[f"{k}|gsq"] = np.float64((grad.astype(np.float64) ** 2).sum())
    np.savez_compressed(os.path.join(HERE, "tiny_step.npz"), **out)
    print("loss", loss.item())


if __name__ == "__main__":
    main()
