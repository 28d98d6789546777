"""Closed-loop calibration: a profiled step timeline -> per
device effective speed in the reference model's units -> calibrated cluster
document -> the reference planner re-plans on it and the executor accepts the
new plan; the in-product cost model prices the executed plan on it."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = os.path.join(ROOT, "configs")
INDEX = json.load(open(os.path.join(CFG, "index.json")))


def docs(name):
    e = INDEX[name]
    return (open(os.path.join(CFG, "clusters", e["cluster"] + ".json")).read(),
            open(os.path.join(CFG, "models", e["model"] + ".json")).read(),
            open(os.path.join(CFG, "plans", name + ".json")).read())


def fake_stats(layer_ms, other_ms, steps):
    # a profiled timeline summed over `steps` steps
    return {"timeline_ms": {
        "gemm_linear": {"ms": 0.8 * layer_ms * steps, "ops": 1},
        "attn_fwd": {"ms": 0.2 * layer_ms * steps, "ops": 1},
        "gemm_lm_head": {"ms": other_ms * steps, "ops": 1},
        "nccl_tp_allreduce": {"ms": 123.0, "ops": 1},
        "step_tick": {"ms": 55.0, "ops": 1}}}


def test_device_speed_counts_layer_work_only():
    from paper_2409_01143_b200 import calibrate
    from paper_2409_01143_b200.hexexec import Plan
    c, m, p = docs("llama7b_4l_tp31")
    L = Plan(c, m, p).layout()
    model = json.loads(m)
    r0, r1 = L["ranks"]
    # rank 0 holds 24/32 heads; 4 layers x 8 micro-batches take 64 ms per step
    st = fake_stats(64.0, 10.0, 2)
    spd = calibrate.device_speed(st, r0, model, 2)
    want = calibrate.layer_flops(model, 1) * 0.75 / (64e-3 / 32)
    assert abs(spd - want) <= 1e-9 * want
    assert calibrate.work_share(r1, model) == 0.25


def test_calibrated_cluster_replans_and_runs_through_the_cost_model():
    from oracle import refshim
    from paper_2409_01143_b200 import calibrate
    from paper_2409_01143_b200.hexexec import Plan
    if not refshim.available():
        pytest.skip("oracle/_ref not built")
    c, m, p = docs("llama7b_4l_4_asym")
    # measured: the two full B200s run at 900 TFLOP/s-equivalent, the halves at 430
    speeds = {"g0": 900e12, "g1": 900e12, "g2": 430e12, "g3": 430e12}
    shares = {"g0": 1.0, "g1": 1.0, "g2": 80 / 148, "g3": 80 / 148}
    cal = calibrate.calibrated_cluster(c, speeds, shares)
    doc = json.loads(cal)
    for d in doc["devices"]:
        assert d["peak_tflops"] == speeds[d["id"]] / 1e12
        assert d["sm_fraction"] == shares[d["id"]]
    # the executor keeps the SM caps it measured under
    L = Plan(cal, m, p).layout()
    assert [r["sm_fraction"] for r in L["ranks"]] == [shares[r["device"]] for r in L["ranks"]]
    # priced on the calibrated speeds (reference formula: equal-speed TP only)
    pred = Plan(cal, m, p).cost(1.0)
    assert pred["feasible"] and pred["total"] > 0
    # re-plan with the reference scheduler on the calibrated cluster; the new
    # plan runs through the executor's parser/layout unchanged
    cfg = json.dumps({"global_batch": 48, "iterations": 30, "seed": 0, "threads": 8,
                      "state_multiplier": 2.5})
    res = refshim.plan(cal, m, cfg, "schedule")
    assert res["found"]
    newL = Plan(cal, m, res["plan"]).layout()
    assert newL["world_size"] == 4
    assert sum(r["samples"][1] - r["samples"][0] for r in newL["ranks"]
               if r["stage"] == 0 and r["tp_index"] == 0) == 48
