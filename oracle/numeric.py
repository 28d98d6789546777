"""ORACLE TEST INFRASTRUCTURE — CPU fp32 restatement of one training step
executed from a HexiScale plan.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg use it, as the checker; the product never does.

The reference has no numeric training step: the step
semantics follow PAPER.md:163-173 (per-pipeline batches, pipeline stages,
DP gradient sync weighted by each pipeline's samples, TP partial sums) and
the payload / FLOP conventions of proj/src/cost_model.cpp:10-128.  The model
math (Llama block: RMSNorm, RoPE, causal MHA, SwiGLU, CE, AdamW) is ours and
defined once in DESIGN.md; this file is its fp32 definition.  Numeric parity
at the reference boundary is therefore *unpinned* by the reference; this
oracle is pinned instead by (a) sharding invariance (sharded == unsharded,
rtol 1e-4) and (b) PyTorch fp32 autograd golden vectors
(tests/golden/make_golden.py).

Execution mirrors the plan: every pipeline runs its own samples; every stage
computes its layers with explicit per-TP-rank partial sums over its own head /
ffn / vocab shards (from oracle/bookkeeping.py); the gradient of the
pipeline's local mean loss is weighted by batch_i / global_batch and summed
over pipelines (the DP allreduce); AdamW updates the global weights.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import bookkeeping as bk
from . import rng

F32 = np.float32
TENSOR_IDS = {"embed": 0, "attn_norm": 1, "wqkv": 2, "wo": 3, "mlp_norm": 4, "wgu": 5,
              "wdown": 6, "final_norm": 7, "lm_head": 8}


def bf16_round(x):
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    x = np.ascontiguousarray(x, dtype=F32)
    u = x.view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000))
    return r.view(F32)


def _ident(x):
    return x



def _pool() -> ThreadPoolExecutor:
    """Host threads for the per-head attention loops and the weight init (numpy
    releases the GIL inside ufuncs / BLAS, so threads scale on the host cores;
    the arithmetic of every element is unchanged)."""
    global _POOL
    if _POOL is None:
        n = int(os.environ.get("HEXEXEC_THREADS", "0")) or (len(os.sched_getaffinity(0))
                                                          if hasattr(os, "sched_getaffinity")
                                                          else os.cpu_count() or 1)
        _POOL = ThreadPoolExecutor(max_workers=max(1, n))
    return _POOL


_POOL = None


def _blas1():
    """One BLAS thread per worker while the per-head pool runs (process-global)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(1, "blas")
    except ImportError:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def init_weights(m: dict, seed: int) -> dict:
    """Global fp32 weights; tensor seed = mix_seed(seed, layer + 1, tensor_id),
    element seed = splitmix64(tensor_seed + global row-major index)."""
    W = {}
    chunk = 1 << 22
    for t in bk.catalogue(m):
        base = t["name"].split(".")[-1]
        if t["kind"] in ("norm", "final_norm"):
            W[t["name"]] = np.ones((t["rows"], t["cols"]), F32)
        else:
            s = rng.mix_seed(seed, t["layer"] + 1, TENSOR_IDS[base])
            n = t["rows"] * t["cols"]
            out = np.empty(n, F32)

            def fill(o, s=s, n=n, out=out):
                out[o:min(n, o + chunk)] = rng.init_normal(s, o, min(chunk, n - o))
            list(_pool().map(fill, range(0, n, chunk)))
            W[t["name"]] = out.reshape(t["rows"], t["cols"])
    return W


def attn_fwd_head(q, k, v, d, rb=_ident):
    """One (sample, head): causal softmax(q k^T / sqrt(d)) v, fp32.  Returns (P, o).
    rb = bf16_round: the un-normalised probabilities enter the PV product as
    bf16 (the fused kernel's P operand), the row sum stays fp32."""
    S = q.shape[0]
    s = (q @ k.T) / F32(np.sqrt(d))
    s = np.where(np.triu(np.ones((S, S), bool), 1), -np.inf, s)
    s = s - s.max(-1, keepdims=True)
    e = np.exp(s)
    l = e.sum(-1, keepdims=True)
    P = (e / l).astype(F32)
    if rb is _ident:
        return P, P @ v
    return P, (rb(e) @ v) / l


def attn_bwd_head(P, q, k, v, dO, d, rb=_ident, o=None):
    """Backward of attn_fwd_head: (dq, dk, dv) before the RoPE inverse.
    rb = bf16_round: delta from the stored bf16 output o, P / dS enter their
    products as bf16 (the fused backward's operands) and dS is formed from the
    bf16 P (the v2 kernel reads P back from shared memory)."""
    Pb = rb(P)
    dV = Pb.T @ dO
    dP = dO @ v.T
    Dv = (P * dP).sum(-1, keepdims=True) if o is None else (dO * o).sum(-1, keepdims=True)
    dS = rb((Pb if rb is not _ident else P) * (dP - Dv) / F32(np.sqrt(d)))
    return dS @ k, dS.T @ q, dV


# ---------------------------------------------------------------- primitives
def rmsnorm(x, g, eps):
    r = (1.0 / np.sqrt((x.astype(np.float64) ** 2).mean(-1, keepdims=True) + eps)).astype(F32)
    return (x * r * g).astype(F32), r


def rmsnorm_bwd(dy, x, r, g):
    H = x.shape[-1]
    xh = x * r
    dg = (dy * xh).sum(0, dtype=np.float64).astype(F32)
    dot = (dy * g * x).sum(-1, keepdims=True, dtype=np.float64).astype(F32)
    dx = r * dy * g - x * (r ** 3) * dot / F32(H)
    return dx.astype(F32), dg


def rope_tables(S, d, theta):
    half = d // 2
    inv = theta ** (-2.0 * np.arange(half, dtype=np.float64) / d)
    ang = np.arange(S, dtype=np.float64)[:, None] * inv[None]
    return np.cos(ang).astype(F32), np.sin(ang).astype(F32)


def rope(x, cos, sin, inverse=False):
    """x [..., S, d] rotate-half; inverse applies the transpose rotation."""
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    s = -sin if inverse else sin
    return np.concatenate([a * cos - b * s, b * cos + a * s], -1).astype(F32)


def silu(x):
    return x / (1.0 + np.exp(-x))



# ---------------------------------------------------------------- model
class Step:
    """One training step of the whole plan (all pipelines) in fp32."""

    def __init__(self, cluster: dict, model: dict, plan_text: str, seed: int = 0,
                 lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1,
                 bf16_points: bool = False):
        """bf16_points: fp32 arithmetic, but every tensor the executor keeps in
        bf16 is rounded to bf16 at the same point (weight copies used by the
        GEMMs, normed inputs, QKV after RoPE, attention P / dS operands and
        output, gate/up, SwiGLU output, final-norm output, dlogits, the bf16
        grads between GEMMs, TP partial sums): the step the executor computes
        up to accumulation order.  False = the plain fp32 definition."""
        self.rb = bf16_round if bf16_points else _ident
        self.m = bk.model_defaults(model)
        self.layout = bk.layout(cluster, model, plan_text)
        self.plan = bk.load_plan(plan_text)
        self.seed = seed
        self.hp = dict(lr=lr, beta1=beta1, beta2=beta2, eps=eps, weight_decay=weight_decay)
        self.W = init_weights(self.m, seed)

    # shard partitions of each stage, from the layout (tp order)
    def stage_parts(self, pipeline: int):
        stages = {}
        for r in self.layout["ranks"]:
            if r["active"] and r["pipeline"] == pipeline:
                stages.setdefault(r["stage"], []).append(r)
        out = []
        for s in sorted(stages):
            rs = sorted(stages[s], key=lambda r: r["tp_index"])
            out.append(dict(layers=tuple(rs[0]["layers"]),
                            parts=[(tuple(r["heads"]), tuple(r["ffn_cols"])) for r in rs],
                            vocab=[tuple(r["vocab_rows"]) for r in rs]))
        return out

    def tokens(self, step: int, sample0: int, n: int):
        return rng.tokens(self.seed, step, sample0, n, self.m["seq_len"], self.m["vocab_size"])

    # -------------------------------------------------------------- forward
    def layer_fwd(self, x, l, parts, mb):
        m, W = self.m, self.W
        S, H, nh = m["seq_len"], m["hidden_dim"], m["num_heads"]
        d = H // nh
        eps = m["norm_eps"]
        p = f"layers.{l}."
        rb, Wb = self.rb, self.Wb
        tp = len(parts) > 1
        c = {"x": x}
        xn, r1 = rmsnorm(x, W[p + "attn_norm"][0], eps)
        xn = rb(xn)
        c.update(xn=xn, r1=r1, parts=[])
        y = np.zeros_like(x)
        cos, sin = rope_tables(S, d, m["rope_theta"])
        for (h0, h1), _ in parts:
            nr = h1 - h0
            qkv = rb(xn @ Wb(p + "wqkv")[3 * d * h0:3 * d * h1].T)       # [M, nr*3*d]
            t = qkv.reshape(mb, S, nr, 3, d).transpose(0, 2, 3, 1, 4)    # [mb, nr, 3, S, d]
            q = rb(rope(t[:, :, 0], cos, sin))
            k = rb(rope(t[:, :, 1], cos, sin))
            v = t[:, :, 2].astype(F32)
            P = np.empty((mb, nr, S, S), F32)
            o = np.empty((mb, nr, S, d), F32)                            # [mb, nr, S, d]

            def head(i):
                b, h = divmod(i, nr)
                P[b, h], o[b, h] = attn_fwd_head(q[b, h], k[b, h], v[b, h], d, rb)
            with _blas1():
                list(_pool().map(head, range(mb * nr)))
            attn = rb(o.transpose(0, 2, 1, 3).reshape(mb * S, nr * d))
            part = attn @ Wb(p + "wo")[d * h0:d * h1]
            y += rb(part) if tp else part
            c["parts"].append(dict(q=q, k=k, v=v, P=P, attn=attn))
        x_mid = (x + y).astype(F32)
        hn, r2 = rmsnorm(x_mid, W[p + "mlp_norm"][0], eps)
        hn = rb(hn)
        c.update(x_mid=x_mid, hn=hn, r2=r2, mparts=[])
        y2 = np.zeros_like(x)
        for _, (f0, f1) in parts:
            gu = rb(hn @ Wb(p + "wgu")[2 * f0:2 * f1].T)
            ch = gu.reshape(-1, (f1 - f0) // 64, 2, 64)
            g = ch[:, :, 0].reshape(-1, f1 - f0)
            u = ch[:, :, 1].reshape(-1, f1 - f0)
            a = rb((silu(g) * u).astype(F32))
            part = a @ Wb(p + "wdown")[f0:f1]
            y2 += rb(part) if tp else part
            c["mparts"].append(dict(g=g, u=u, a=a))
        return (x_mid + y2).astype(F32), c

    def Wb(self, name):
        """The weight copy the GEMMs read (bf16 points: the bf16 copy)."""
        if self.rb is _ident:
            return self.W[name]
        if getattr(self, "_wb_src", None) is not self.W:
            self._wb_src, self._wb = self.W, {}
        if name not in self._wb:
            self._wb[name] = bf16_round(self.W[name])
        return self._wb[name]

    def layer_bwd(self, dx_out, l, parts, c, mb, G):
        m, W = self.m, self.W
        S, H, nh = m["seq_len"], m["hidden_dim"], m["num_heads"]
        d = H // nh
        p = f"layers.{l}."
        cos, sin = rope_tables(S, d, m["rope_theta"])
        rb, Wb = self.rb, self.Wb
        bf = rb is not _ident
        dxo = rb(dx_out)                    # the bf16 copy the GEMMs read
        dhn = np.zeros_like(dx_out)
        for (_, (f0, f1)), mp in zip(parts, c["mparts"]):
            Wd = Wb(p + "wdown")[f0:f1]
            G[p + "wdown"][f0:f1] += mp["a"].T @ dxo
            da = rb(dxo @ Wd.T)
            sg = 1.0 / (1.0 + np.exp(-mp["g"]))
            dg = da * mp["u"] * sg * (1.0 + mp["g"] * (1.0 - sg))
            du = da * mp["g"] * sg
            n = (f1 - f0) // 64
            dgu = rb(np.stack([dg.reshape(-1, n, 64), du.reshape(-1, n, 64)], 2)
                     .reshape(-1, 2 * (f1 - f0)).astype(F32))
            G[p + "wgu"][2 * f0:2 * f1] += dgu.T @ c["hn"]
            dhn += rb(dgu @ Wb(p + "wgu")[2 * f0:2 * f1])
        dxm, dg2 = rmsnorm_bwd(dhn.astype(F32), c["x_mid"], c["r2"], W[p + "mlp_norm"][0])
        G[p + "mlp_norm"][0] += dg2
        dx_mid = (dx_out + dxm).astype(F32)
        dxmb = rb(dx_mid)
        dxn = np.zeros_like(dx_out)
        for ((h0, h1), _), ap in zip(parts, c["parts"]):
            nr = h1 - h0
            G[p + "wo"][d * h0:d * h1] += ap["attn"].T @ dxmb
            dattn = rb(dxmb @ Wb(p + "wo")[d * h0:d * h1].T)
            dO = dattn.reshape(mb, S, nr, d).transpose(0, 2, 1, 3)
            oo = ap["attn"].reshape(mb, S, nr, d).transpose(0, 2, 1, 3) if bf else None
            dq = np.empty((mb, nr, S, d), F32)
            dk = np.empty((mb, nr, S, d), F32)
            dV = np.empty((mb, nr, S, d), F32)

            def head(i, ap=ap, dO=dO, dq=dq, dk=dk, dV=dV, oo=oo):
                b, h = divmod(i, nr)
                dq[b, h], dk[b, h], dV[b, h] = attn_bwd_head(
                    ap["P"][b, h], ap["q"][b, h], ap["k"][b, h], ap["v"][b, h],
                    np.ascontiguousarray(dO[b, h]), d, rb,
                    None if oo is None else np.ascontiguousarray(oo[b, h]))
            with _blas1():
                list(_pool().map(head, range(mb * nr)))
            dq = rb(rope(rb(dq), cos, sin, inverse=True))
            dk = rb(rope(rb(dk), cos, sin, inverse=True))
            dqkv = rb(np.stack([dq, dk, dV], 2).transpose(0, 3, 1, 2, 4).reshape(mb * S, nr * 3 * d))
            G[p + "wqkv"][3 * d * h0:3 * d * h1] += dqkv.T @ c["xn"]
            dxn += rb(dqkv @ Wb(p + "wqkv")[3 * d * h0:3 * d * h1])
        dxi, dg1 = rmsnorm_bwd(dxn.astype(F32), c["x"], c["r1"], W[p + "attn_norm"][0])
        G[p + "attn_norm"][0] += dg1
        return (dx_mid + dxi).astype(F32)

    def micro_batch(self, tok, stages, count, G):
        """fwd + bwd of one micro-batch (tok [mb, S+1]); grads of
        sum(CE)/count accumulated into G; returns the CE sum."""
        m, W = self.m, self.W
        mb, S = tok.shape[0], m["seq_len"]
        inp, tgt = tok[:, :S].reshape(-1), tok[:, 1:].reshape(-1)
        x = W["embed"][inp].astype(F32)
        caches = []
        for st in stages:                       # PP hand-off is the identity in-process
            for l in range(*st["layers"]):
                x, c = self.layer_fwd(x, l, st["parts"], mb)
                caches.append((l, st["parts"], c))
        last = stages[-1]
        rb = self.rb
        xf, rf = rmsnorm(x, W["final_norm"][0], m["norm_eps"])
        xf = rb(xf)
        logits = np.concatenate([xf @ self.Wb("lm_head")[v0:v1].T for v0, v1 in last["vocab"]], -1)
        mx = logits.max(-1, keepdims=True)
        e = np.exp((logits - mx).astype(np.float64))
        se = e.sum(-1, keepdims=True)
        loss = float((np.log(se[:, 0]) + mx[:, 0] - logits[np.arange(len(tgt)), tgt]).sum())
        dl = (e / se).astype(F32)
        dl[np.arange(len(tgt)), tgt] -= 1.0
        dl *= F32(1.0 / count)
        dl = rb(dl)
        G["lm_head"] += dl.T @ xf
        if len(last["vocab"]) > 1 and rb is not _ident:   # TP partials of the dgrad, bf16
            dxf = sum(rb(dl[:, v0 - last["vocab"][0][0]:v1 - last["vocab"][0][0]]
                         @ self.Wb("lm_head")[v0:v1]) for v0, v1 in last["vocab"])
        else:
            dxf = rb(dl @ self.Wb("lm_head"))
        dx, dgf = rmsnorm_bwd(dxf.astype(F32), x, rf, W["final_norm"][0])
        G["final_norm"][0] += dgf
        for l, parts, c in reversed(caches):
            dx = self.layer_bwd(dx, l, parts, c, mb, G)
        np.add.at(G["embed"], inp, dx)
        return loss

    def run(self, step: int = 0):
        """One optimizer step.  Returns (global mean loss, reduced grads, new W)."""
        m = self.m
        S = m["seq_len"]
        B = self.plan["global_batch"]
        total = {k: np.zeros_like(v) for k, v in self.W.items()}
        loss_sum = 0.0
        s0 = 0
        for pi, p in enumerate(self.plan["pipelines"]):
            stages = self.stage_parts(pi)
            G = {k: np.zeros_like(v) for k, v in self.W.items()}
            toks = self.tokens(step, s0, p["batch"])
            for i in range(p["batch"] // p["micro_batch"]):
                t = toks[i * p["micro_batch"]:(i + 1) * p["micro_batch"]]
                loss_sum += self.micro_batch(t, stages, p["batch"] * S, G)
            w = F32(p["batch"] / B)             # DP weight of this pipeline
            for k in total:
                total[k] += w * G[k]
            s0 += p["batch"]
        self.grads = total
        self.adamw(total, step + 1)
        return loss_sum / (B * S), total, self.W

    def adamw(self, G, t):
        hp = self.hp
        if not hasattr(self, "mom"):
            self.mom = {k: np.zeros_like(v) for k, v in self.W.items()}
            self.vel = {k: np.zeros_like(v) for k, v in self.W.items()}
        b1, b2 = F32(hp["beta1"]), F32(hp["beta2"])
        bc1, bc2 = F32(1 - hp["beta1"] ** t), F32(1 - hp["beta2"] ** t)
        for k, g in G.items():
            kind = k.split(".")[-1]
            wd = 0.0 if kind in ("attn_norm", "mlp_norm", "final_norm") else hp["weight_decay"]
            self.mom[k] = b1 * self.mom[k] + (1 - b1) * g
            self.vel[k] = b2 * self.vel[k] + (1 - b2) * g * g
            upd = (self.mom[k] / bc1) / (np.sqrt(self.vel[k] / bc2) + F32(hp["eps"]))
            self.W[k] = (self.W[k] - F32(hp["lr"]) * (upd + F32(wd) * self.W[k])).astype(F32)
