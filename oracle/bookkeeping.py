"""ORACLE TEST INFRASTRUCTURE — integer plan bookkeeping, restated in Python.

Used only by tests/ (and bench.py's cpu_baseline leg) as the checker of the
executor's C++ bookkeeping (paper_2409_01143_b200/csrc/plan.cpp).

Reference semantics restated here:
  * PipelinePlan::num_micro_batches     /root/reference/proj/src/types.hpp:70-72
  * build_dp_groups                     /root/reference/proj/src/cost_model.cpp:155-164
  * validate_plan (same messages)       /root/reference/proj/src/cost_model.cpp:166-208
  * plan wire format                    /root/reference/proj/src/report.cpp:25-53
and pinned against the compiled reference itself (oracle/_ref/libhexplan_ref.so,
see oracle/refshim.py) and the reference's own test vectors
(proj/tests/test_cost_model.cpp:294-361).

Extensions (not in the reference): tp_widths,
largest-remainder shard split of heads / 64-col ffn chunks / 64-row vocab
chunks, sample ranges, PP peers, chunk-matched DP buckets.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field


class InvalidArgument(Exception):
    pass


def load_plan(text: str) -> dict:
    j = json.loads(text)
    if isinstance(j, dict) and isinstance(j.get("plan"), dict):
        j = j["plan"]  # CLI artifact {"manifest":..., "plan":...}
    return j


def model_defaults(m: dict) -> dict:
    H = m["hidden_dim"]
    out = dict(m)
    out.setdefault("num_heads", H // 128 if H % 128 == 0 else H // 64)
    f = (8 * H + 2) // 3
    out.setdefault("ffn_dim", (f + 255) // 256 * 256)
    out.setdefault("vocab_size", 32000)
    out.setdefault("rope_theta", 10000.0)
    out.setdefault("norm_eps", 1e-5)
    return out


def build_dp_groups(plan: dict, num_layers: int, dev_index) -> list:
    """cost_model.cpp:155-164: per layer, the first device of the hosting stage
    of every pipeline, in pipeline order."""
    groups = [{"layer": l, "members": []} for l in range(num_layers)]
    for p in plan["pipelines"]:
        for st in p["stages"]:
            if not st["devices"]:
                continue
            for l in range(st["layer_start"], st["layer_start"] + st["layer_count"]):
                if 0 <= l < num_layers:
                    groups[l]["members"].append(st["devices"][0])
    return groups


def validate_plan(plan: dict, num_layers: int, n_devices: int, dev_index) -> None:
    """cost_model.cpp:166-208, same checks in the same order, same messages."""
    P = plan["pipelines"]
    if not P:
        raise InvalidArgument("plan has no pipelines")
    if plan["global_batch"] < 1:
        raise InvalidArgument("plan has no batch")
    used = [False] * n_devices
    batch_sum = 0
    for p in P:
        if not p["stages"]:
            raise InvalidArgument("pipeline has no stages")
        if p["micro_batch"] < 1 or p["batch"] < p["micro_batch"]:
            raise InvalidArgument("pipeline batch smaller than its micro batch")
        if p["batch"] % p["micro_batch"] != 0:
            raise InvalidArgument("pipeline batch not a micro batch multiple")
        batch_sum += p["batch"]
        nxt = 0
        for st in p["stages"]:
            if not st["devices"]:
                raise InvalidArgument("stage has no devices")
            if st["tp"] != len(st["devices"]):
                raise InvalidArgument("stage tp degree does not match its device count")
            if st["layer_count"] < 1:
                raise InvalidArgument("stage holds no layers")
            if st["layer_start"] != nxt:
                raise InvalidArgument("stages do not tile the layer range")
            nxt += st["layer_count"]
            for d in st["devices"]:
                i = dev_index(d)
                if i < 0 or i >= n_devices:
                    raise InvalidArgument("stage references an unknown device")
                if used[i]:
                    raise InvalidArgument("device appears in two stages")
                used[i] = True
        if nxt != num_layers:
            raise InvalidArgument("pipeline does not cover all layers")
    if batch_sum != plan["global_batch"]:
        raise InvalidArgument("pipeline batches do not sum to the global batch")
    g = plan["dp_groups"]
    if len(g) != num_layers:
        raise InvalidArgument("dp groups do not cover all layers")
    for l, grp in enumerate(g):
        if grp["layer"] != l:
            raise InvalidArgument("dp group layer index out of order")
        if len(grp["members"]) != len(P):
            raise InvalidArgument("dp group missing a pipeline replica")


def num_micro_batches(p: dict) -> int:
    """types.hpp:70-72 (C++ integer division of positive values)."""
    return p["batch"] // p["micro_batch"] if p["micro_batch"] > 0 else 0


def largest_remainder(units: int, weights: list[int]) -> list[int]:
    """Exact-integer Hamilton apportionment; ties -> lower index."""
    W = sum(weights)
    q = [units * w for w in weights]
    out = [x // W for x in q]
    rem = sorted(range(len(weights)), key=lambda i: (-(q[i] % W), i))
    for k in range(units - sum(out)):
        out[rem[k]] += 1
    return out


TENSORS = ["attn_norm", "wqkv", "wo", "mlp_norm", "wgu", "wdown"]


def catalogue(m: dict) -> list[dict]:
    H, F, V, L = m["hidden_dim"], m["ffn_dim"], m["vocab_size"], m["num_layers"]
    t = [dict(name="embed", layer=-1, kind="embed", rows=V, cols=H)]
    for l in range(L):
        p = f"layers.{l}."
        t += [dict(name=p + "attn_norm", layer=l, kind="norm", rows=1, cols=H),
              dict(name=p + "wqkv", layer=l, kind="wqkv", rows=3 * H, cols=H),
              dict(name=p + "wo", layer=l, kind="wo", rows=H, cols=H),
              dict(name=p + "mlp_norm", layer=l, kind="norm", rows=1, cols=H),
              dict(name=p + "wgu", layer=l, kind="wgu", rows=2 * F, cols=H),
              dict(name=p + "wdown", layer=l, kind="wdown", rows=F, cols=H)]
    t += [dict(name="final_norm", layer=-1, kind="final_norm", rows=1, cols=H),
          dict(name="lm_head", layer=-1, kind="lm_head", rows=V, cols=H)]
    return t


@dataclass
class Role:
    rank: int
    device: str
    active: bool = False
    pipeline: int = -1
    stage: int = -1
    stage_count: int = 1
    tp_index: int = 0
    tp: int = 1
    layers: tuple = (0, 0)
    heads: tuple = (0, 0)
    ffn_cols: tuple = (0, 0)
    vocab_rows: tuple = (0, 0)
    samples: tuple = (0, 0)
    micro_batch: int = 0
    num_micro_batches: int = 0
    tp_group: list = field(default_factory=list)
    fwd_recv_from: int = -1
    bwd_recv_from: int = -1
    fwd_send_to: list = field(default_factory=list)
    bwd_send_to: list = field(default_factory=list)
    dp_weight: float = 1.0
    tensors: list = field(default_factory=list)  # dicts name,row0,rows,cols,offset,multiplicity


def layout(cluster: dict, model: dict, plan_text: str) -> dict:
    """Integer layout of every world rank (mirrors hexexec_plan_layout_json)."""
    m = model_defaults(model)
    plan = load_plan(plan_text)
    devs = cluster["devices"]
    ids = [d["id"] for d in devs]

    def dev_index(x):
        if isinstance(x, str):
            return ids.index(x) if x in ids else -1
        return x

    plan = json.loads(json.dumps(plan))
    for p in plan["pipelines"]:
        for st in p["stages"]:
            st["devices"] = [dev_index(d) for d in st["devices"]]
    if "dp_groups" in plan:
        for g in plan["dp_groups"]:
            g["members"] = [dev_index(d) for d in g["members"]]
    else:
        plan["dp_groups"] = build_dp_groups(plan, m["num_layers"], dev_index)
    validate_plan(plan, m["num_layers"], len(devs), lambda i: i)

    n = len(devs)
    rank_of = [d.get("rank", i) for i, d in enumerate(devs)]
    maxp = max(d["peak_tflops"] for d in devs)
    roles = [None] * n
    for i, d in enumerate(devs):
        roles[rank_of[i]] = Role(rank=rank_of[i], device=d["id"])
    H, F, V, nh_total = m["hidden_dim"], m["ffn_dim"], m["vocab_size"], m["num_heads"]
    dh = H // nh_total
    off = 0
    for pi, p in enumerate(plan["pipelines"]):
        for sj, st in enumerate(p["stages"]):
            w = st.get("tp_widths") or [1] * st["tp"]
            if len(w) != st["tp"]:
                raise InvalidArgument("stage tp_widths length does not match its device count")
            heads = largest_remainder(nh_total, w)
            ffn = largest_remainder(F // 64, w)
            voc = largest_remainder(V // 64, w)
            group = [rank_of[d] for d in st["devices"]]
            h0 = f0 = v0 = 0
            for t in range(st["tp"]):
                if heads[t] < 1:
                    raise InvalidArgument("tp shard holds no attention heads")
                if ffn[t] < 1:
                    raise InvalidArgument("tp shard holds no ffn columns")
                if voc[t] < 1:
                    raise InvalidArgument("tp shard holds no vocab rows")
                r = roles[group[t]]
                r.active = True
                r.pipeline, r.stage, r.stage_count = pi, sj, len(p["stages"])
                r.tp_index, r.tp = t, st["tp"]
                r.layers = (st["layer_start"], st["layer_start"] + st["layer_count"])
                r.heads = (h0, h0 + heads[t])
                r.ffn_cols = (64 * f0, 64 * (f0 + ffn[t]))
                r.vocab_rows = (64 * v0, 64 * (v0 + voc[t]))
                h0 += heads[t]
                f0 += ffn[t]
                v0 += voc[t]
                r.samples = (off, off + p["batch"])
                r.micro_batch = p["micro_batch"]
                r.num_micro_batches = num_micro_batches(p)
                r.tp_group = group
                r.dp_weight = p["batch"] / plan["global_batch"]
                if sj > 0:
                    prev = p["stages"][sj - 1]
                    r.fwd_recv_from = rank_of[prev["devices"][t % prev["tp"]]]
                    r.bwd_send_to = [rank_of[prev["devices"][u]] for u in range(prev["tp"])
                                     if u % st["tp"] == t]
                if sj + 1 < len(p["stages"]):
                    nx = p["stages"][sj + 1]
                    r.bwd_recv_from = rank_of[nx["devices"][t % nx["tp"]]]
                    r.fwd_send_to = [rank_of[nx["devices"][u]] for u in range(nx["tp"])
                                     if u % st["tp"] == t]
        off += p["batch"]

    cat = catalogue(m)
    for r in roles:
        o = 0
        if not r.active:
            continue
        for t in cat:
            held = (r.layers[0] <= t["layer"] < r.layers[1]) if t["layer"] >= 0 else (
                r.stage == 0 if t["kind"] == "embed" else r.stage == r.stage_count - 1)
            if not held:
                continue
            k = t["kind"]
            row0, rows, mult = 0, t["rows"], 1
            if k in ("embed", "norm", "final_norm"):
                mult = r.tp
            elif k == "wqkv":
                row0, rows = 3 * dh * r.heads[0], 3 * dh * (r.heads[1] - r.heads[0])
            elif k == "wo":
                row0, rows = dh * r.heads[0], dh * (r.heads[1] - r.heads[0])
            elif k == "wgu":
                row0, rows = 2 * r.ffn_cols[0], 2 * (r.ffn_cols[1] - r.ffn_cols[0])
            elif k == "wdown":
                row0, rows = r.ffn_cols[0], r.ffn_cols[1] - r.ffn_cols[0]
            elif k == "lm_head":
                row0, rows = r.vocab_rows[0], r.vocab_rows[1] - r.vocab_rows[0]
            r.tensors.append(dict(name=t["name"], row0=row0, rows=rows, cols=t["cols"],
                                  offset=o, multiplicity=mult))
            o += rows * t["cols"]

    # communicator sets + chunk-matched DP buckets
    sets, set_idx = [], {}

    def intern(s):
        s = tuple(sorted(s))
        if s not in set_idx:
            set_idx[s] = len(sets)
            sets.append(list(s))
        return set_idx[s]

    tp_comm = [-1] * n
    for r in roles:
        if r.active and r.tp > 1:
            tp_comm[r.rank] = intern(r.tp_group)
    segs = []
    for t in cat:
        cols = t["cols"]
        # sync group: layer index, -1 embedding, -2 head (final norm + LM head)
        group = t["layer"] if t["layer"] >= 0 else (-1 if t["kind"] == "embed" else -2)
        hs, cuts = [], set()
        for r in roles:
            for rt in r.tensors:
                if rt["name"] == t["name"]:
                    b, e = rt["row0"] * cols, (rt["row0"] + rt["rows"]) * cols
                    hs.append((r.rank, b, e, rt["offset"]))
                    cuts.update([b, e])
        cuts = sorted(cuts)
        for a, b in zip(cuts, cuts[1:]):
            ranks = [(h[0], h[3] + a - h[1]) for h in hs if h[1] <= a and b <= h[2]]
            if len(ranks) >= 2 and b > a:
                segs.append(([x[0] for x in ranks], [x[1] for x in ranks], b - a, group))
    merged = []
    for sg in segs:
        if merged:
            mr, ml, mlen, mg = merged[-1]
            if mr == sg[0] and mg == sg[3] and all(ml[i] + mlen == sg[1][i] for i in range(len(mr))):
                merged[-1] = (mr, ml, mlen + sg[2], mg)
                continue
        merged.append(sg)
    buckets = [[] for _ in range(n)]
    for ranks, locs, ln, grp in merged:
        ci = intern(ranks)
        for rk, lo in zip(ranks, locs):
            buckets[rk].append({"comm": ci, "offset": lo, "count": ln, "group": grp})

    out_ranks = []
    for r in roles:
        jr = {"rank": r.rank, "device": r.device, "active": r.active}
        if r.active:
            jr.update(pipeline=r.pipeline, stage=r.stage, tp_index=r.tp_index, tp=r.tp,
                      layers=list(r.layers), heads=list(r.heads), ffn_cols=list(r.ffn_cols),
                      vocab_rows=list(r.vocab_rows), samples=list(r.samples),
                      micro_batch=r.micro_batch, num_micro_batches=r.num_micro_batches,
                      tp_group=r.tp_group, tp_comm=tp_comm[r.rank],
                      fwd_recv_from=r.fwd_recv_from, bwd_recv_from=r.bwd_recv_from,
                      fwd_send_to=r.fwd_send_to, bwd_send_to=r.bwd_send_to,
                      dp_weight=r.dp_weight,
                      param_count=sum(t["rows"] * t["cols"] for t in r.tensors),
                      tensors=r.tensors, dp_buckets=buckets[r.rank])
        out_ranks.append(jr)
    return {
        "world_size": n,
        "num_micro_batches": [num_micro_batches(p) for p in plan["pipelines"]],
        "dp_groups": [{"layer": g["layer"], "members": [ids[i] for i in g["members"]]}
                      for g in plan["dp_groups"]],
        "comm_sets": sets,
        "ranks": out_ranks,
    }
