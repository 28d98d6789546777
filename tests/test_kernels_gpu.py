"""Kernel-level parity: each sm_100a kernel (called through the C ABI) against a
plain PyTorch fp32 reference of the same op on the same inputs.

Tolerances: GEMMs accumulate in fp32 on bf16 inputs, so they are compared to
an fp32 matmul of the same bf16 values at rtol 2e-3 of the output scale; bf16
outputs add one bf16 rounding (2^-8).  Memory-bound kernels in fp32: rtol 1e-4.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _L():
    from paper_2409_01143_b200 import _lib
    return _lib


def _ptr(t):
    return None if t is None else t.data_ptr()


def _gemm(A, a_mn, B, b_mn, M, N, K, C, *, beta=0, alpha=1.0, causal=0, nb1=1, nb2=1,
          a_bs=(0, 0), b_bs=(0, 0), c_bs=(0, 0), lda=None, ldb=None, ldc=None):
    L = _L()
    lda = lda if lda is not None else (M if a_mn else K)
    ldb = ldb if ldb is not None else (N if b_mn else K)
    ldc = ldc if ldc is not None else N
    st = L.hexexec_k_gemm(M, N, K, nb1, nb2, _ptr(A), a_mn, lda, a_bs[0], a_bs[1], _ptr(B), b_mn,
                          ldb, b_bs[0], b_bs[1], _ptr(C), ldc, c_bs[0], c_bs[1],
                          1 if C.dtype == torch.float32 else 0, beta, alpha, causal, None)
    assert st == 0
    torch.cuda.synchronize()


def _rel(out, ref):
    return (out.float() - ref.float()).abs().max().item() / max(ref.float().abs().max().item(), 1e-30)


@pytest.mark.parametrize("split", [-1, 2, 3, 5])
@pytest.mark.parametrize("M,N,K,a_mn,b_mn", [(2048, 4096, 1024, 0, 1), (512, 1024, 512, 1, 1),
                                             (384, 704, 640, 0, 0)])
def test_gemm_tail_split(cuda, split, M, N, K, a_mn, b_mn):
    """Split-K of the partial last wave: bf16 / fp32 stores go through the
    fp32 workspace (last partial finishes the tile), beta GEMMs reduce-add
    partials into C; workspace and counters must be left zero."""
    L = _L()
    ws = torch.zeros(148 * 128 * 256, device=cuda)
    cnt = torch.zeros(148 * 8, device=cuda, dtype=torch.int32)
    assert L.hexexec_k_gemm_split(split, ws.data_ptr(), ws.numel() * 4, cnt.data_ptr(),
                                  cnt.numel()) == 0
    try:
        g = torch.Generator(device="cuda").manual_seed(M + N + K)
        A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
        B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
        ref = A.float() @ B.float().T
        As = A.T.contiguous() if a_mn else A
        Bs = B.T.contiguous() if b_mn else B
        for _ in range(2):  # second call checks the workspace was left clean
            C16 = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
            _gemm(As, a_mn, Bs, b_mn, M, N, K, C16)
            assert _rel(C16, ref) < 1e-2
            C32 = torch.zeros(M, N, device=cuda)
            _gemm(As, a_mn, Bs, b_mn, M, N, K, C32, alpha=0.5)
            assert _rel(C32, 0.5 * ref) < 2e-3
            acc = torch.ones(M, N, device=cuda)
            _gemm(As, a_mn, Bs, b_mn, M, N, K, acc, beta=1)
            assert _rel(acc, ref + 1) < 2e-3
        assert ws.abs().max().item() == 0.0
        assert cnt.abs().max().item() == 0
    finally:
        L.hexexec_k_gemm_split(-1, None, 0, None, 0)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (384, 192, 192), (128, 2752, 128),
                                   (304, 200, 96)])
def test_gemm_layouts(cuda, a_mn, b_mn, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    ref = A.float() @ B.float().T
    As = A.T.contiguous() if a_mn else A
    Bs = B.T.contiguous() if b_mn else B
    C32 = torch.zeros(M, N, device=cuda)
    _gemm(As, a_mn, Bs, b_mn, M, N, K, C32)
    assert _rel(C32, ref) < 2e-3
    C16 = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
    _gemm(As, a_mn, Bs, b_mn, M, N, K, C16)
    assert _rel(C16, ref) < 1e-2


def test_gemm_beta_alpha(cuda):
    M, N, K = 256, 384, 320
    A = torch.randn(M, K, device=cuda).bfloat16()
    B = torch.randn(N, K, device=cuda).bfloat16()
    C = torch.randn(M, N, device=cuda)
    ref = C + 0.5 * (A.float() @ B.float().T)
    _gemm(A, 0, B, 0, M, N, K, C, beta=1, alpha=0.5)
    assert _rel(C, ref) < 2e-3


def test_gemm_large_tp_shapes(cuda):
    # Llama-7B shard shapes: QKV 3:1 col shard (N=9216) and down-proj K tail (2752)
    for (M, N, K) in [(2048, 9216, 4096), (2048, 4096, 2752)]:
        A = torch.randn(M, K, device=cuda).bfloat16()
        B = torch.randn(N, K, device=cuda).bfloat16()
        C = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
        _gemm(A, 0, B, 0, M, N, K, C)
        ref = A.float() @ B.float().T
        assert _rel(C, ref) < 1e-2


def test_gemm_batched_heads(cuda):
    # per-(sample, head) scores straight out of the fused [M, nh*3*d] QKV buffer
    mb, S, nh, d = 2, 256, 3, 64
    qkv = torch.randn(mb * S, nh * 3 * d, device=cuda).bfloat16()
    W = nh * 3 * d
    out = torch.zeros(mb, nh, S, S, device=cuda)
    q = qkv.view(mb, S, nh, 3, d)[:, :, :, 0]
    k = qkv.view(mb, S, nh, 3, d)[:, :, :, 1]
    _gemm(qkv, 0, qkv[:, d:], 0, S, S, d, out, nb1=nh, nb2=mb, lda=W, ldb=W,
          a_bs=(3 * d, S * W), b_bs=(3 * d, S * W), c_bs=(S * S, nh * S * S), alpha=0.125)
    ref = torch.einsum("bshd,bthd->bhst", q.float(), k.float()) * 0.125
    assert _rel(out, ref) < 2e-3


def test_gemm_causal_modes(cuda):
    L_, d = 384, 64
    Q = torch.randn(L_, d, device=cuda).bfloat16()
    K = torch.randn(L_, d, device=cuda).bfloat16()
    # skip-upper: every entry on/below the diagonal is computed; whole output
    # tiles (128 x BN) strictly above it are skipped and left untouched
    S = torch.full((L_, L_), 7.0, device=cuda)
    _gemm(Q, 0, K, 0, L_, L_, d, S, causal=1)
    ref = Q.float() @ K.float().T
    lower = torch.ones(L_, L_, device=cuda).tril().bool()
    assert _rel(S[lower], ref[lower]) < 2e-3
    assert torch.all(S[:128, 256:] == 7.0)  # tile (m0=0, n0=256) skipped
    # k-lower: lower-triangular A (P) times V
    P = torch.tril(torch.rand(L_, L_, device=cuda)).bfloat16()
    V = torch.randn(L_, d, device=cuda).bfloat16()
    O = torch.zeros(L_, d, device=cuda)
    _gemm(P, 0, V, 1, L_, d, L_, O, causal=2)  # B = V^T logically [d, L], stored MN-major
    assert _rel(O, P.float() @ V.float()) < 2e-3
    # k-upper: dV = P^T dO, A = P^T stored MN-major (P itself)
    dO = torch.randn(L_, d, device=cuda).bfloat16()
    dV = torch.zeros(L_, d, device=cuda)
    _gemm(P, 1, dO, 1, L_, d, L_, dV, causal=3)
    assert _rel(dV, P.float().T @ dO.float()) < 2e-3


def test_rmsnorm_fwd_bwd(cuda):
    L = _L()
    M, H, eps = 64, 512, 1e-5
    x = torch.randn(M, H, device=cuda)
    y = torch.randn(M, H, device=cuda).bfloat16()
    g = torch.rand(H, device=cuda) + 0.5
    xo = torch.empty_like(x)
    out = torch.empty(M, H, device=cuda, dtype=torch.bfloat16)
    rstd = torch.empty(M, device=cuda)
    assert L.hexexec_k_rmsnorm_fwd(_ptr(x), _ptr(y), _ptr(xo), _ptr(g), _ptr(out), _ptr(rstd),
                                   M, H, eps, None) == 0
    torch.cuda.synchronize()
    xs = x + y.float()
    r = torch.rsqrt(xs.pow(2).mean(-1, keepdim=True) + eps)
    assert torch.allclose(xo, xs, rtol=1e-6, atol=1e-6)
    assert torch.allclose(rstd, r[:, 0], rtol=1e-4)
    assert _rel(out, xs * r * g) < 1e-2
    # backward with fp32 dy and residual grad
    dy = torch.randn(M, H, device=cuda)
    dres = torch.randn(M, H, device=cuda)
    dx = torch.empty_like(x)
    dxb = torch.empty(M, H, device=cuda, dtype=torch.bfloat16)
    dg = torch.zeros(H, device=cuda)
    assert L.hexexec_k_rmsnorm_bwd(None, _ptr(dy), _ptr(xs), _ptr(rstd), _ptr(g), _ptr(dres),
                                   _ptr(dx), _ptr(dxb), _ptr(dg), M, H, None) == 0
    torch.cuda.synchronize()
    xr = xs.clone().requires_grad_(True)
    gr = g.clone().requires_grad_(True)
    yy = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + eps) * gr
    yy.backward(dy)
    assert torch.allclose(dx, xr.grad + dres, rtol=1e-4, atol=1e-4)
    assert torch.allclose(dg, gr.grad, rtol=1e-4, atol=1e-3)
    assert _rel(dxb, xr.grad + dres) < 1e-2


def _rope_ref(x, pos, theta, inverse=False):
    d = x.shape[-1]
    half = d // 2
    inv = theta ** (-2.0 * torch.arange(half, device=x.device, dtype=torch.float64) / d)
    ang = pos[:, None].double() * inv[None]
    c, s = torch.cos(ang).float(), torch.sin(ang).float()
    if inverse:
        s = -s
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * c[:, None] - b * s[:, None], b * c[:, None] + a * s[:, None]], -1)


def test_rope_roundtrip(cuda):
    L = _L()
    mb, S, nh, d = 2, 128, 3, 64
    M = mb * S
    qkv = torch.randn(M, nh * 3 * d, device=cuda).bfloat16()
    orig = qkv.clone()
    assert L.hexexec_k_rope(_ptr(qkv), M, S, nh, d, 10000.0, 0, None) == 0
    torch.cuda.synchronize()
    pos = torch.arange(M, device=cuda) % S
    v = orig.view(M, nh, 3, d).float()
    got = qkv.view(M, nh, 3, d).float()
    assert _rel(got[:, :, 0], _rope_ref(v[:, :, 0], pos, 10000.0)) < 1e-2
    assert _rel(got[:, :, 1], _rope_ref(v[:, :, 1], pos, 10000.0)) < 1e-2
    assert torch.equal(got[:, :, 2], v[:, :, 2])


def test_softmax_fwd_bwd(cuda):
    L = _L()
    nb, L_ = 3, 256
    S = torch.randn(nb, L_, L_, device=cuda)
    P = torch.full((nb, L_, L_), 9.0, device=cuda).bfloat16()
    assert L.hexexec_k_softmax_fwd(_ptr(S), _ptr(P), L_, nb, None) == 0
    torch.cuda.synchronize()
    mask = torch.ones(L_, L_, device=cuda).tril().bool()
    ref = torch.softmax(S.masked_fill(~mask, float("-inf")), -1)
    lower = mask.expand(nb, L_, L_)
    assert _rel(P.float()[lower], ref[lower]) < 1e-2
    # zeros inside the diagonal tile, untouched beyond it
    i = 5
    assert torch.all(P[:, i, i + 1:128].float() == 0)
    assert torch.all(P[:, i, 128:].float() == 9.0)
    dP = torch.randn(nb, L_, L_, device=cuda)
    dS = torch.zeros(nb, L_, L_, device=cuda).bfloat16()
    assert L.hexexec_k_softmax_bwd(_ptr(P), _ptr(dP), _ptr(dS), 0.5, L_, nb, None) == 0
    torch.cuda.synchronize()
    Pf = P.float().masked_fill(~mask, 0)
    Dv = (Pf * dP).sum(-1, keepdim=True)
    refd = 0.5 * Pf * (dP - Dv)
    assert _rel(dS.float()[lower], refd[lower]) < 2e-2


def test_swiglu(cuda):
    L = _L()
    M, F = 64, 192
    gu = torch.randn(M, 2 * F, device=cuda).bfloat16()
    a = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
    assert L.hexexec_k_swiglu_fwd(_ptr(gu), _ptr(a), M, F, None) == 0
    v = gu.float().view(M, F // 64, 2, 64)
    g, u = v[:, :, 0].reshape(M, F), v[:, :, 1].reshape(M, F)
    gr, ur = g.clone().requires_grad_(True), u.clone().requires_grad_(True)
    out = torch.nn.functional.silu(gr) * ur
    torch.cuda.synchronize()
    assert _rel(a, out) < 1e-2
    da = torch.randn(M, F, device=cuda).bfloat16()
    dgu = torch.empty(M, 2 * F, device=cuda, dtype=torch.bfloat16)
    assert L.hexexec_k_swiglu_bwd(_ptr(gu), _ptr(da), _ptr(dgu), M, F, None) == 0
    torch.cuda.synchronize()
    out.backward(da.float())
    dv = dgu.float().view(M, F // 64, 2, 64)
    assert _rel(dv[:, :, 0].reshape(M, F), gr.grad) < 1e-2
    assert _rel(dv[:, :, 1].reshape(M, F), ur.grad) < 1e-2


def test_cross_entropy(cuda):
    L = _L()
    mb, S, V = 2, 128, 512
    M = mb * S
    logits = torch.randn(M, V, device=cuda) * 3
    tok = torch.randint(0, V, (mb, S + 1), device=cuda, dtype=torch.int32)
    dl = torch.empty(M, V, device=cuda, dtype=torch.bfloat16)
    loss = torch.zeros(1, device=cuda)
    scratch = torch.empty(5 * M, device=cuda)
    inv = 1.0 / M
    assert L.hexexec_k_ce(_ptr(logits), V, 0, _ptr(tok), M, S, inv, _ptr(dl), _ptr(loss),
                          _ptr(scratch), None) == 0
    torch.cuda.synchronize()
    tgt = tok[:, 1:].reshape(-1).long()
    lr = logits.clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lr, tgt, reduction="sum")
    ref.backward()
    assert abs(loss.item() - ref.item()) / ref.item() < 1e-4
    assert _rel(dl, lr.grad * inv) < 1e-2


def test_adamw(cuda):
    L = _L()
    n = 10000
    p = torch.randn(n, device=cuda)
    m = torch.randn(n, device=cuda) * 0.01
    v = torch.rand(n, device=cuda) * 0.01
    g = torch.randn(n, device=cuda)
    p16 = torch.empty(n, device=cuda, dtype=torch.bfloat16)
    p0, m0, v0 = p.clone(), m.clone(), v.clone()
    lr, b1, b2, eps, wd, step = 1e-3, 0.9, 0.95, 1e-8, 0.1, 3
    assert L.hexexec_k_adamw(_ptr(p), _ptr(p16), _ptr(m), _ptr(v), None, _ptr(g), n, 0.5, lr, b1,
                             b2, eps, wd, step, None) == 0
    torch.cuda.synchronize()
    gg = g * 0.5
    mr = b1 * m0 + (1 - b1) * gg
    vr = b2 * v0 + (1 - b2) * gg * gg
    mh = mr / (1 - b1 ** step)
    vh = vr / (1 - b2 ** step)
    pr = p0 - lr * (mh / (vh.sqrt() + eps) + wd * p0)
    assert torch.allclose(m, mr, rtol=1e-5, atol=1e-7)
    assert torch.allclose(v, vr, rtol=1e-5, atol=1e-9)
    assert torch.allclose(p, pr, rtol=1e-4, atol=1e-6)
    assert torch.equal(p16, p.bfloat16())


def test_init_and_tokens_match_oracle(cuda):
    from oracle import rng as O
    L = _L()
    n, off, seed = 5000, 123456, 987654321
    out = torch.empty(n, device=cuda)
    assert L.hexexec_k_init_normal(_ptr(out), n, off, seed, None) == 0
    torch.cuda.synchronize()
    ref = O.init_normal(seed, off, n)
    assert np.array_equal(out.cpu().numpy(), ref)  # bit-exact
    ns, S, s0, step, V = 3, 64, 5, 2, 512
    tok = torch.empty(ns, S + 1, device=cuda, dtype=torch.int32)
    assert L.hexexec_k_tokens(_ptr(tok), ns, S, s0, 7, step, V, None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(tok.cpu().numpy(), O.tokens(7, step, s0, ns, S, V))


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(512, 1024, 256), (256, 768, 192), (2048, 4096, 1024),
                                   (384, 1280, 320)])
def test_gemm_a_multicast(cuda, a_mn, b_mn, M, N, K):
    """Clusters of two CTA pairs along N sharing the A tile via TMA multicast
    (odd N-tile counts leave the second pair of the last cluster out of range)."""
    L = _L()
    assert L.hexexec_k_gemm_multicast(2) == 0
    try:
        g = torch.Generator(device="cuda").manual_seed(M + N * 3 + K)
        A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
        B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
        ref = A.float() @ B.float().T
        As = A.T.contiguous() if a_mn else A
        Bs = B.T.contiguous() if b_mn else B
        C16 = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
        _gemm(As, a_mn, Bs, b_mn, M, N, K, C16)
        assert _rel(C16, ref) < 1e-2
        C32 = torch.randn(M, N, device=cuda)
        ref2 = C32 + ref
        _gemm(As, a_mn, Bs, b_mn, M, N, K, C32, beta=1)
        assert _rel(C32, ref2) < 2e-3
    finally:
        assert L.hexexec_k_gemm_multicast(1) == 0
