"""bench.py helpers (CPU): the nvidia-smi sampler keeps only rows inside the
timed window and reports per-GPU medians, the delivered SM-GHz, and the
reference-convention FLOP count (cost_model.cpp:17-21, :260-265)."""
import datetime
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_clocks_window_and_per_gpu():
    ck = bench.Clocks(2)
    t0 = datetime.datetime(2026, 1, 1, 12, 0, 0)
    rows = []
    for i in range(10):
        ts = (t0 + datetime.timedelta(milliseconds=100 * i)).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        for g, mhz in (("0", 1500 + i), ("1", 1965)):
            rows.append(f"{ts}, {g}, {mhz}, 1965, 900.0, 0x4, Not Active, Not Active, Not Active, "
                        f"{'Active' if g == '0' else 'Not Active'}")
    ck.f.write("\n".join(rows) + "\n")
    ck.f.flush()
    ck.p = type("P", (), {"terminate": lambda s: None, "wait": lambda s: 0})()
    ck.t0 = t0 + datetime.timedelta(milliseconds=250)
    ck.t1 = t0 + datetime.timedelta(milliseconds=750)
    out = ck.stop()
    assert out["samples"] == 10  # 5 timestamps x 2 GPUs inside the window
    assert out["sm_mhz_per_gpu"] == {"0": 1505.0, "1": 1965.0}
    assert out["reasons"] == ["sw_power_cap"]
    assert out["gpu_of_rank"] == ["0", "1"]


def test_sm_ghz_and_flops():
    r = {"clocks": {"sm_mhz_per_gpu": {"0": 1500.0, "1": 1965.0}, "gpu_of_rank": ["0", "1"]},
         "lin_per_rank": [[0, 0, 0, 1.0], [0, 0, 0, 56 / 148]]}
    assert abs(bench.sm_ghz(r) - (148 * 1.5 + 56 * 1.965)) < 1e-9
    c, m, p, _ = bench.load("llama7b_4l_1gpu")
    md = bench.full_model(c, m, p)
    ref, exact = bench.model_flops(md, 2048)
    L, H, S = md["num_layers"], md["hidden_dim"], md["seq_len"]
    assert abs(ref - 72.0 * 2048 * H * H * (1 + S / (6.0 * H)) * L) / ref < 1e-12
    assert exact > ref  # exact counts the LM head and the non-causal-free GEMMs


def test_default_plans_exist():
    idx = json.load(open(os.path.join(ROOT, "configs", "index.json")))
    for n, (asym, even) in bench.PLANS.items():
        assert asym in idx
        for e in (even or "").split(","):
            assert not e or e in idx
    for n, names in bench.ALT.items():
        for a in names.split(","):
            assert a in idx


def test_cpu_reference_bounded_sample(monkeypatch):
    """The reference arm's unit: one sample through the whole model when it has
    at most MAX_REF_LAYERS layers (nothing extrapolated); deeper models run the
    first MAX_REF_LAYERS layers and label the FLOP-ratio extrapolation.  Only
    oracle code runs (no product library)."""
    r = bench.cpu_reference("tiny_1", steps=1, warmup=0)
    assert r["kind"] == "port" and r["value"] > 0 and "extrapolation" not in r
    assert r["ms_per_sample"] > 0 and len(r["sample_ms"]) == 1
    monkeypatch.setattr(bench, "MAX_REF_LAYERS", 2)
    r2 = bench.cpu_reference("tiny_1", steps=1, warmup=0)
    ex = r2["extrapolation"]
    assert ex["layers_run"] == 2 and ex["layers"] == 4 and 0 < ex["training_flop_ratio"] < 1
    assert abs(r2["value"] - ex["measured_unit_tokens_per_s"] * ex["training_flop_ratio"]) < 1e-6


def test_summarize_delivered_clock_mfu():
    """MFU at delivered clock = reference FLOPs / (sum SMs x median clock x 8192)."""
    c, m, p, _ = bench.load("llama7b_4l_1gpu")
    r = {"name": "llama7b_4l_1gpu", "plan": json.loads(p), "model": json.loads(m),
         "cluster": json.loads(c), "dev_ms": 1000.0, "e2e_ms": 1000.0, "sm_share": 1.0,
         "loss": 1.0, "clocks": {"sm_mhz_per_gpu": {"0": 1500.0}, "gpu_of_rank": ["0"]},
         "lin_per_rank": [[0, 0, 0, 1.0]]}
    s = bench.summarize(r, steps=10, pk={"bf16_tflops": 1646.0})
    md = bench.full_model(c, m, p)
    ref, _ = bench.model_flops(md, 8 * 2048)
    assert abs(s["mfu_at_delivered_clock"] - ref / 0.1 / (148 * 1.5 * 8192e9)) < 1e-9
    assert abs(s["mfu_ref_convention"] - ref / 0.1 / 1646e12) < 1e-9
