"""Integer plan bookkeeping: product (C ABI) vs Python oracle vs compiled reference.

Bit-exact: num_micro_batches (types.hpp:70-72), dp_groups (cost_model.cpp:155-164),
validate_plan messages (cost_model.cpp:166-208), plan serialization
(report.cpp:25-64), and the extension layout (shards, samples, PP peers,
chunk-matched DP buckets).  No GPU needed.
"""
import ctypes as C
import glob
import json
import os
import re

import pytest

from oracle import bookkeeping as bk
from oracle import refshim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = os.path.join(ROOT, "configs")
INDEX = json.load(open(os.path.join(CFG, "index.json")))


def docs(name):
    e = INDEX[name]
    c = open(os.path.join(CFG, "clusters", e["cluster"] + ".json")).read()
    m = open(os.path.join(CFG, "models", e["model"] + ".json")).read()
    p = open(os.path.join(CFG, "plans", name + ".json")).read()
    return c, m, p


# the reference's own C-ABI test inputs (proj/tests/test_capi.cpp:11-29)
TOY_CLUSTER = json.dumps({
    "machines": {"A": {"intra_bandwidth_gbps": 200, "intra_latency_us": 10},
                 "B": {"intra_bandwidth_gbps": 32, "intra_latency_us": 500}},
    "devices": [{"id": "a0", "machine": "A", "memory_gib": 80, "peak_tflops": 312},
                {"id": "a1", "machine": "A", "memory_gib": 80, "peak_tflops": 312},
                {"id": "b0", "machine": "B", "memory_gib": 24, "peak_tflops": 165},
                {"id": "b1", "machine": "B", "memory_gib": 24, "peak_tflops": 165}],
    "inter": {"bandwidth_gbps": 12, "latency_us": 1000}})
TOY_MODEL = json.dumps({"num_layers": 8, "hidden_dim": 2048, "seq_len": 2048,
                        "bytes_per_element": 2})
# golden plan of hexplan_schedule on the toy inputs (seed 1, 1 thread)
TOY_PLAN = json.dumps({"global_batch": 16, "pipelines": [
    {"batch": 8, "micro_batch": 1, "num_micro_batches": 8, "stages": [
        {"devices": ["b0"], "tp": 1, "layer_start": 0, "layer_count": 2},
        {"devices": ["a0"], "tp": 1, "layer_start": 2, "layer_count": 6}]},
    {"batch": 8, "micro_batch": 1, "num_micro_batches": 8, "stages": [
        {"devices": ["b1"], "tp": 1, "layer_start": 0, "layer_count": 2},
        {"devices": ["a1"], "tp": 1, "layer_start": 2, "layer_count": 6}]}],
    "dp_groups": [{"layer": l, "members": ["b0", "b1"] if l < 2 else ["a0", "a1"]}
                  for l in range(8)]})


def product():
    from paper_2409_01143_b200 import _lib as L
    from paper_2409_01143_b200.hexexec import Plan
    return L, Plan


def test_library_exports_every_header_symbol():
    L, _ = product()
    hdr = open(os.path.join(ROOT, "include", "hexexec.h")).read()
    names = set(re.findall(r"\b(hexexec_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L.lib, n)]
    assert not missing, missing
    assert set(L.EXPORTED) == names


ALL = sorted(INDEX)


@pytest.mark.parametrize("name", ALL)
def test_layout_matches_python_oracle(name):
    _, Plan = product()
    c, m, p = docs(name)
    got = Plan(c, m, p).layout()
    want = bk.layout(json.loads(c), json.loads(m), p)
    for k in ("world_size", "num_micro_batches", "dp_groups", "comm_sets"):
        assert got[k] == want[k], k
    for gr, wr in zip(got["ranks"], want["ranks"]):
        for k, v in wr.items():
            assert gr[k] == v, (gr["rank"], k)


@pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ALL)
def test_bookkeeping_matches_compiled_reference(name):
    _, Plan = product()
    c, m, p = docs(name)
    ref = refshim.check_plan(c, m, p)
    assert ref["validate"] == "ok"
    lay = Plan(c, m, p).layout()
    assert lay["num_micro_batches"] == ref["num_micro_batches"]
    assert lay["dp_groups"] == ref["dp_groups"]


@pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ALL)
def test_serialize_is_byte_identical_to_reference(name):
    _, Plan = product()
    c, m, p = docs(name)
    ref = refshim.check_plan(c, m, p)
    assert Plan(c, m, p).serialize() == ref["plan_serialized"]
    if INDEX[name]["source"].startswith("hexplan_"):
        assert Plan(c, m, p).serialize() == p  # committed planner output, verbatim


def test_wrapped_cli_plan_is_accepted():
    _, Plan = product()
    c, m, p = docs("tiny_dp53")
    wrapped = json.dumps({"manifest": {"version": "hexplan 0.1.0", "command": "schedule",
                                       "inputs": [], "seed": 0, "config": {}},
                          "plan": json.loads(p)})
    assert Plan(c, m, wrapped).layout() == Plan(c, m, p).layout()


def test_reference_dp_group_kat():
    """proj/tests/test_cost_model.cpp:341-361: members {2,0},{2,0},{4,0},{4,0}."""
    _, Plan = product()
    cl = json.dumps({"machines": {"m": {"intra_bandwidth_gbps": 16, "intra_latency_us": 0}},
                     "devices": [{"id": f"d{i}", "machine": "m", "memory_gib": 80,
                                  "peak_tflops": 100} for i in range(5)],
                     "inter": {"bandwidth_gbps": 16, "latency_us": 0}})
    md = json.dumps({"num_layers": 4, "hidden_dim": 2048, "seq_len": 2048,
                     "bytes_per_element": 2})
    plan = {"global_batch": 2, "pipelines": [
        {"batch": 1, "micro_batch": 1, "stages": [
            {"devices": ["d2", "d3"], "tp": 2, "layer_start": 0, "layer_count": 2},
            {"devices": ["d4"], "tp": 1, "layer_start": 2, "layer_count": 2}]},
        {"batch": 1, "micro_batch": 1, "stages": [
            {"devices": ["d0", "d1"], "tp": 2, "layer_start": 0, "layer_count": 4}]}]}
    want = [["d2", "d0"], ["d2", "d0"], ["d4", "d0"], ["d4", "d0"]]
    lay = Plan(cl, md, json.dumps(plan)).layout()
    assert [g["members"] for g in lay["dp_groups"]] == want
    py = bk.layout(json.loads(cl), json.loads(md), json.dumps(plan))
    assert [g["members"] for g in py["dp_groups"]] == want
    if refshim.available():
        ref = refshim.check_plan(cl, md, json.dumps(plan))
        assert [g["members"] for g in ref["dp_groups"]] == want


def _violations():
    """proj/tests/test_cost_model.cpp:294-339 plus the remaining validate_plan
    checks, as plan-document edits of a good 2-pipeline plan."""
    def good():
        return {"global_batch": 4, "pipelines": [
            {"batch": 2, "micro_batch": 1, "stages": [
                {"devices": ["d0"], "tp": 1, "layer_start": 0, "layer_count": 8}]},
            {"batch": 2, "micro_batch": 1, "stages": [
                {"devices": ["d1"], "tp": 1, "layer_start": 0, "layer_count": 8}]}],
            "dp_groups": [{"layer": l, "members": ["d0", "d1"]} for l in range(8)]}
    cases = []
    p = good(); p["pipelines"][1]["stages"][0]["devices"] = ["d0"]; cases.append(("reuse", p))
    p = good(); p["pipelines"][0]["stages"][0]["layer_count"] = 7; cases.append(("cover", p))
    p = good(); p["pipelines"][0]["stages"][0]["tp"] = 2; cases.append(("tp", p))
    p = good(); p["global_batch"] = 5; cases.append(("batch", p))
    p = good(); p["pipelines"][0]["micro_batch"] = 3; cases.append(("micro", p))
    p = good(); p["dp_groups"].pop(); cases.append(("dpgroups", p))
    p = good(); p["pipelines"] = []; cases.append(("nopipes", p))
    p = good(); p["global_batch"] = 0; cases.append(("nobatch", p))
    p = good(); p["pipelines"][0]["stages"] = []; cases.append(("nostages", p))
    p = good(); p["pipelines"][0]["micro_batch"] = 4; p["pipelines"][0]["batch"] = 2; cases.append(("small", p))
    p = good(); p["pipelines"][0]["stages"][0]["devices"] = []; p["pipelines"][0]["stages"][0]["tp"] = 0; cases.append(("nodev", p))
    p = good(); p["pipelines"][0]["stages"][0]["layer_count"] = 0; cases.append(("nolayers", p))
    p = good(); p["pipelines"][0]["stages"][0]["layer_start"] = 1; cases.append(("tile", p))
    p = good(); p["pipelines"][0]["stages"][0]["devices"] = [7]; cases.append(("unknown", p))
    p = good(); p["dp_groups"][3]["layer"] = 5; cases.append(("order", p))
    p = good(); p["dp_groups"][3]["members"] = ["d0"]; cases.append(("replica", p))
    return cases


@pytest.mark.parametrize("tag,plan", _violations())
def test_validate_plan_messages_match_reference(tag, plan):
    L, Plan = product()
    from paper_2409_01143_b200.hexexec import HexexecError
    cl = json.dumps({"machines": {"m": {"intra_bandwidth_gbps": 16, "intra_latency_us": 0}},
                     "devices": [{"id": f"d{i}", "machine": "m", "memory_gib": 80,
                                  "peak_tflops": 100} for i in range(3)],
                     "inter": {"bandwidth_gbps": 16, "latency_us": 0}})
    md = json.dumps({"num_layers": 8, "hidden_dim": 2048, "seq_len": 2048,
                     "bytes_per_element": 2})
    with pytest.raises(HexexecError) as ei:
        Plan(cl, md, json.dumps(plan))
    assert ei.value.status == L.ERR_INVALID
    with pytest.raises(bk.InvalidArgument) as ej:
        bk.layout(json.loads(cl), json.loads(md), json.dumps(plan))
    assert ei.value.msg == str(ej.value)
    if refshim.available():
        ref = refshim.check_plan(cl, md, json.dumps(plan))
        assert ref["validate"] == ei.value.msg


def test_toy_reference_plan_and_mixed_type_stage():
    _, Plan = product()
    lay = Plan(TOY_CLUSTER, TOY_MODEL, TOY_PLAN).layout()
    assert lay["num_micro_batches"] == [8, 8]
    # hand plan the reference cost model cannot price (TP over full + 1/3 devices)
    if refshim.available():
        c, m, p = docs("llama7b_4l_tp31")
        ref = refshim.check_plan(c, m, p)
        assert ref["validate"] == "ok"
        assert ref.get("cost_error") == "mixed-type tensor parallel stage"


def test_error_conventions():
    L, Plan = product()
    err = C.create_string_buffer(8)
    h = C.c_void_p()
    assert L.hexexec_plan_parse(None, b"{}", b"{}", C.byref(h), err, len(err)) == L.ERR_INVALID
    assert err.value == b"null ar"  # truncated, NUL-terminated (capi.cpp:34-39)
    c, m, p = docs("tiny_1")
    assert L.hexexec_plan_parse(c.encode(), m.encode(), b"{not json", C.byref(h), err,
                                len(err)) == L.ERR_PARSE
    assert L.hexexec_plan_parse(b"[]", m.encode(), p.encode(), C.byref(h), None, 0) == L.ERR_PARSE
    # extension checks: widths length, shard without heads
    bad = json.loads(p)
    bad["pipelines"][0]["stages"][0]["tp_widths"] = [1, 1]
    big = C.create_string_buffer(256)
    assert L.hexexec_plan_parse(c.encode(), m.encode(), json.dumps(bad).encode(), C.byref(h),
                                big, len(big)) == L.ERR_INVALID
    assert b"tp_widths" in big.value


def test_exec_config_is_strict_and_no_cpu_path():
    L, _ = product()
    c, m, p = docs("tiny_1")
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    st = L.hexexec_ctx_create(c.encode(), m.encode(), p.encode(), b'{"bogus": 1}', 0, 1, 0,
                              None, 0, C.byref(h), err, len(err))
    assert st == L.ERR_PARSE and b"unknown key" in err.value
    st = L.hexexec_ctx_create(c.encode(), m.encode(), p.encode(), b'{"validate_only": true}', 0,
                              1, 0, None, 0, C.byref(h), err, len(err))
    assert st == L.OK
    L.hexexec_ctx_free(h)
    import torch
    if not torch.cuda.is_available():
        st = L.hexexec_ctx_create(c.encode(), m.encode(), p.encode(), b"{}", 0, 1, 0, None, 0,
                                  C.byref(h), err, len(err))
        assert st == L.ERR_CUDA, err.value


def test_shard_rules():
    assert bk.largest_remainder(32, [3, 1]) == [24, 8]
    assert bk.largest_remainder(172, [3, 1]) == [129, 43]      # 11008 / 64 -> 8256 / 2752
    assert bk.largest_remainder(4, [3, 1]) == [3, 1]
    assert bk.largest_remainder(5, [1, 1, 1]) == [2, 2, 1]     # ties -> lower index
    assert bk.largest_remainder(40, [2, 2, 1]) == [16, 16, 8]
    _, Plan = product()
    c, m, p = docs("llama7b_4l_tp31")
    r = Plan(c, m, p).layout()["ranks"]
    assert r[0]["heads"] == [0, 24] and r[1]["heads"] == [24, 32]
    assert r[0]["ffn_cols"] == [0, 8256] and r[1]["ffn_cols"] == [8256, 11008]


@pytest.mark.parametrize("cfg,ok", [
    ('{"pp_dtype": "bf16"}', True), ('{"pp_dtype": "fp32"}', True), ('{"pp_dtype": "fp16"}', False),
    ('{"attention": "unfused", "recompute": true}', True), ('{"tp_reduce": "ring"}', False),
    ('{"wgrad_group": "x"}', False), ('{"dp_comm_dtype": "fp32", "tp_pull": "sm"}', True),
])
def test_exec_config_values(cfg, ok):
    """Every exec-config key of include/hexexec.h validates its value at the
    boundary (strict like the reference's config parser, json_io.cpp:263)."""
    L, _ = product()
    c, m, p = docs("tiny_1")
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    full = json.dumps(dict(json.loads(cfg), validate_only=True))
    st = L.hexexec_ctx_create(c.encode(), m.encode(), p.encode(), full.encode(), 0, 1, 0, None, 0,
                              C.byref(h), err, len(err))
    if ok:
        assert st == L.OK, err.value
        L.hexexec_ctx_free(h)
    else:
        assert st == L.ERR_PARSE, (st, err.value)


def test_head_dim_256_layout_and_large_micro_batch_sizing():
    """Host side of the size-limit rows: a head_dim 256 model and a 20480-token
    micro-batch both size their arena host-only (validate_only), and the
    head_dim 256 plan reports the unfused attention path."""
    L, _ = product()
    for name in ("tiny_d256_1", "tiny_bigmb"):
        c, m, p = docs(name)
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        st = L.hexexec_ctx_create(c.encode(), m.encode(), p.encode(), b'{"validate_only": true}', 0,
                                  1, 0, None, 0, C.byref(h), err, len(err))
        assert st == L.OK, (name, err.value)
        stats = json.loads(L.take_string(L.hexexec_stats_json(h)))
        L.hexexec_ctx_free(h)
        assert stats["arena_bytes"] > 0
        if name == "tiny_d256_1":
            assert stats["attention"].startswith("unfused"), stats["attention"]
