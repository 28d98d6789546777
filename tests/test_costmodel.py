"""The executor's restatement of the reference cost model
(csrc/costmodel.cpp <- proj/src/cost_model.cpp:10-265) against
(1) the compiled reference itself on every BASELINE config (identical report
JSON, identical refusal of mixed-speed TP stages) and (2) the known-answer
vectors of the reference's own tests (test_cost_model.cpp), expressed as
cluster / model / plan documents through the C ABI."""
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


@pytest.mark.parametrize("name", sorted(INDEX))
def test_report_equals_compiled_reference(name):
    from oracle import refshim
    from paper_2409_01143_b200.hexexec import HexexecError, Plan
    if not refshim.available():
        pytest.skip("oracle/_ref not built")
    c, m, p = docs(name)
    ref = refshim.check_plan(c, m, p)
    plan = Plan(c, m, p)
    if "cost" in ref:
        assert plan.cost(1.0) == ref["cost"]
    else:
        with pytest.raises(HexexecError) as ei:
            plan.cost(1.0)
        assert ref["cost_error"] in str(ei.value)
    # the extension prices every plan, and equals the reference where it applies
    ext = plan.cost(1.0, extension=True)
    assert ext["feasible"] and ext["total"] > 0
    if "cost" in ref and all(
            not json.loads(p)["pipelines"][i]["stages"][j].get("tp_widths")
            for i in range(len(json.loads(p)["pipelines"]))
            for j in range(len(json.loads(p)["pipelines"][i]["stages"]))):
        assert ext == ref["cost"]


def flat(flops, beta_gbs, alpha_us, names=None):
    n = len(flops)
    return json.dumps({
        "machines": {"m": {"intra_bandwidth_gbps": beta_gbs, "intra_latency_us": alpha_us}},
        "devices": [{"id": f"d{i}", "machine": "m", "memory_gib": 1e9, "peak_tflops": f / 1e12}
                    for i, f in enumerate(flops)],
        "inter": {"bandwidth_gbps": beta_gbs, "latency_us": alpha_us}})


def model(L, H, S, B=2):
    return json.dumps({"num_layers": L, "hidden_dim": H, "seq_len": S, "bytes_per_element": B})


def one_pipeline(stages, batch=1, mb=1):
    return json.dumps({"global_batch": batch, "pipelines": [{
        "batch": batch, "micro_batch": mb, "stages": [
            {"devices": d, "tp": len(d), "layer_start": a, "layer_count": n} for d, a, n in stages]}]})


def cost(c, m, p):
    from paper_2409_01143_b200.hexexec import Plan
    return Plan(c, m, p).cost(1.0)


def rel_close(got, want, tol=1e-9):
    return abs(got - want) <= tol * abs(want)


def test_kat_compute_time_and_mfu():
    # test_cost_model.cpp "per-layer compute time": 1 + S/6H == 2, c = 1236950581248
    r = cost(flat([1236950581248.0], 1, 0), model(1, 1024, 6144), one_pipeline([(["d0"], 0, 1)]))
    assert rel_close(r["compute"], 1.0) and rel_close(r["total"], 1.0)
    assert rel_close(r["mfu"], 0.75)
    # 2048 / 2048 at 1e14 FLOP/s: 9.62072674304e-3 s
    r = cost(flat([1e14], 1, 0), model(1, 2048, 2048), one_pipeline([(["d0"], 0, 1)]))
    assert rel_close(r["compute"], 9.62072674304e-3)


def test_kat_tp_allreduce():
    # "tensor parallel allreduce time": 0.012582912 (alpha 0), 0.013782912 (alpha 100 us)
    for alpha, want in ((0, 0.012582912), (100, 0.013782912)):
        r = cost(flat([1e12, 1e12], 16, alpha), model(1, 4096, 4096),
                 one_pipeline([(["d0", "d1"], 0, 1)]))
        assert rel_close(r["tp_comm"], want)


def test_kat_dp_sync():
    # "data parallel sync time": 2 members 0.402653184, 3 members 0.536870912
    for n, want in ((2, 0.402653184), (3, 0.536870912)):
        p = json.dumps({"global_batch": n, "pipelines": [
            {"batch": 1, "micro_batch": 1,
             "stages": [{"devices": [f"d{i}"], "tp": 1, "layer_start": 0, "layer_count": 1}]}
            for i in range(n)]})
        r = cost(flat([1e12] * 3, 1, 0), model(1, 4096, 4096), p)
        assert rel_close(r["dp_comm"], want)


def test_kat_pipeline_hop():
    # "pipeline hop time": 0.067308864 (beta 1 GB/s, alpha 100 us)
    r = cost(flat([1e12, 1e12], 1, 100), model(2, 4096, 4096),
             one_pipeline([(["d0"], 0, 1), (["d1"], 1, 1)]))
    assert rel_close(r["pp_comm"], 0.067308864)


def test_mixed_tp_refused_like_reference_and_priced_by_extension():
    from paper_2409_01143_b200.hexexec import HexexecError, Plan
    c = flat([1e14, 2e14], 1000, 0)
    m = model(1, 2048, 2048)
    p = json.loads(one_pipeline([(["d0", "d1"], 0, 1)]))
    plan = Plan(c, m, json.dumps(p))
    with pytest.raises(HexexecError, match="mixed-type tensor parallel stage"):
        plan.cost(1.0)
    # equal widths: the slower rank (1e14) does half the FLOPs
    fl = 96 * 2048 * 2048 * 2048 * (1 + 2048 / (6 * 2048))
    assert rel_close(plan.cost(1.0, extension=True)["compute"], 0.5 * fl / 1e14)
    # widths 1:2 match the speeds: both ranks take a third of the FLOPs at their rate
    p["pipelines"][0]["stages"][0]["tp_widths"] = [1, 2]
    plan = Plan(c, m, json.dumps(p))
    assert rel_close(plan.cost(1.0, extension=True)["compute"], fl / 3 / 1e14)
