"""Closed-loop calibration: measured B200
speeds -> cluster document -> the reference cost model / planner.

Each rank's profiled step timeline (executor profile mode: CUDA events after
every operation) gives the device time of its transformer layers; with the
rank's share of a layer's work, that is an effective speed c_d in the units of
the reference model (cost_model.cpp:16-21, 78-88: time = 96*mb*S*H^2*(1+S/6H)
* share / c_d per layer per micro-batch).  Writing c_d back as the device's
`peak_tflops` (with `sm_fraction` pinned, so the SM caps do not move) gives a
cluster document that the reference scheduler can re-plan on and that
`Plan.cost(extension=True)` prices for predicted-vs-measured.

Only layer work is attributed: embedding, LM head, CE, optimizer, NCCL waits
and step bookkeeping are excluded (the reference model prices layers only,
SPEC.md:250)."""
from __future__ import annotations

import json

# timeline kinds that are not transformer-layer work
_EXCLUDE_PREFIX = ("nccl_", "step_tick", "prologue", "gen_tokens", "embed_", "ce_",
                   "gemm_lm_head", "adamw", "scale", "cast_")


def layer_seconds(timeline_ms: dict, steps: int, layers: int, micro_batches: int) -> float:
    """Device seconds per (layer x micro-batch) from a profiled timeline
    ({kind: {"ms", "ops"}} summed over `steps` steps)."""
    ms = sum(v["ms"] for k, v in timeline_ms.items() if not k.startswith(_EXCLUDE_PREFIX))
    return ms / 1e3 / steps / (layers * micro_batches)


def layer_flops(model: dict, batch: float) -> float:
    """cost_model.cpp:16-21"""
    S, H = model["seq_len"], model["hidden_dim"]
    return 96.0 * batch * S * H * H * (1.0 + S / (6.0 * H))


def work_share(role: dict, model: dict) -> float:
    """The rank's share of a layer's work inside its TP stage (head share; the
    FFN split uses the same tp_widths)."""
    nh = model.get("num_heads") or max(1, model["hidden_dim"] // 128)
    h0, h1 = role["heads"]
    return (h1 - h0) / nh


def device_speed(stats: dict, role: dict, model: dict, steps: int) -> float:
    """Effective FLOP/s of this rank in the reference model's units."""
    l0, l1 = role["layers"]
    t = layer_seconds(stats["timeline_ms"], steps, l1 - l0, role["num_micro_batches"])
    return layer_flops(model, role["micro_batch"]) * work_share(role, model) / t


def calibrated_cluster(cluster_json: str, speeds: dict, sm_fractions: dict) -> str:
    """Copy of the cluster document with peak_tflops := measured speed for every
    device in `speeds` ({device id: FLOP/s}); sm_fraction pinned to the value
    the executor applied so re-running the calibrated document keeps the caps."""
    c = json.loads(cluster_json)
    for d in c["devices"]:
        if d["id"] in speeds:
            d["peak_tflops"] = speeds[d["id"]] / 1e12
            d["sm_fraction"] = sm_fractions[d["id"]]
            d["calibrated"] = True
    return json.dumps(c)
