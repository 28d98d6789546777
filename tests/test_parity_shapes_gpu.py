"""GPU-vs-oracle parity at the benchmarked shapes (VERDICT r01 "What's
missing" 1-2): the full step (fwd, bwd, sample-weighted DP sync, AdamW)
through the C ABI compared with the CPU fp32 oracle (oracle/numeric.py) on
the same seeds and tokens -- loss, every reduced gradient, every updated
weight, rtol 2e-2 normwise (BASELINE north star: bf16 tensor-core
accumulation vs the fp32 oracle).

* llama7b_2l_1gpu: the headline workload's layer shape (H 4096, 32 heads,
  d 128, F 11008, V 32000, S 2048 = 16 attention key tiles), 2 layers,
  2 micro-batches (weight-gradient accumulation), one B200, in-process.
* llama7b_2l_tp31: the same on 2 GPUs with TP widths 3:1 and the second
  rank SM-capped to 1/3 (cfg2's shards: heads 24/8, FFN 8256/2752 with a
  64-column K tail, vocab 24000/8000), TP partials over NVLink peer memory.
* 13B / 30B layer shapes at S 256 (H 5120 / 6656, 40 / 52 heads, F 13824 /
  17920): one B200 and TP 3:1 (heads 30/10, 39/13).
* 4-GPU analogues of cfg4 and of a mixed plan at 13B layer shapes:
  3-stage PP 2/1/1 with an uneven TP stage (3:1 over a full and a
  half-capped B200), and TP 2:1 + PP + DP 3:2 with mismatched TP degrees
  (chunk-matched DP buckets).

Bars (see _check): at these shapes any two bf16 implementations of the
step differ from the fp32 definition by 3-4 % normwise on the gradients
(PyTorch's bf16 autocast step on the same weights / tokens: 3.3 % at the 7B
shape, 3.5 % at 13B), because the activations and gradients are *stored* in
bf16 between the GEMMs.  So the gradients are held to 2e-2 against the
oracle with the executor's bf16 storage points emulated, and to PyTorch's
bf16 deviation against the plain fp32 oracle.  The fp32 oracle itself is
pinned at these shapes by an independent fp32 PyTorch autograd restatement
(test_oracle_pinned_by_torch_fp32, rtol 1e-4).

Large-shape oracles are not cached (several GB per copy); a summary of the
errors per tensor is printed (pytest -s) for the logs in profiles/.
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity_util import (RTOL, ngpu, oracle_for, rel, run_inprocess, run_plan,  # noqa: E402
                         torch_floor, world_of)


def _check(name, ranks):
    """Three references for the same step: the fp32 oracle, the oracle with
    the executor's bf16 storage points (bf16_points), and PyTorch's bf16
    autocast step (the bf16 floor).  Asserted, per tensor:
      * loss within RTOL (2e-2) of the fp32 oracle;
      * updated weight within RTOL of the fp32 oracle and of the bf16-points
        oracle;
      * gradient deviation from the fp32 oracle <= 1.25 x PyTorch bf16's own
        deviation (+2e-3): as close to the fp32 definition as a standard bf16
        mixed-precision step gets at this shape (measured: 0.97-1.00 x);
      * gradient deviation from the bf16-points oracle <= max(RTOL, the bf16
        floor): with the rounding points emulated, what remains is
        accumulation order and the decorrelation of later roundings, which
        grows with depth (1.8 % at 2 layers, 3.1 % at 4 layers of 13B)."""
    loss, G, W = oracle_for(name, keep=False)
    tloss, floor = torch_floor(name, G)
    ours_g, ours_w = {}, {}
    for r in ranks:
        for key in r:
            if key.endswith("|grad"):
                t = key[:-5]
                row0 = int(r[t + "|row0"])
                n = r[key].shape[0]
                ours_g[t] = max(ours_g.get(t, 0.0), rel(r[key], G[t][row0:row0 + n]))
                ours_w[t] = max(ours_w.get(t, 0.0), rel(r[t + "|w"], W[t][row0:row0 + n]))
    del G, W
    eloss, Ge, We = oracle_for(name, keep=False, bf16_points=True)
    emu_g, emu_w = {}, {}
    for r in ranks:
        for key in r:
            if key.endswith("|grad"):
                t = key[:-5]
                row0 = int(r[t + "|row0"])
                n = r[key].shape[0]
                emu_g[t] = max(emu_g.get(t, 0.0), rel(r[key], Ge[t][row0:row0 + n]))
                emu_w[t] = max(emu_w.get(t, 0.0), rel(r[t + "|w"], We[t][row0:row0 + n]))
    held = set(ours_g)
    rows = {t: [round(ours_g[t], 5), round(floor[t], 5), round(emu_g[t], 5), round(ours_w[t], 5),
                round(emu_w[t], 5)] for t in sorted(held)}
    print("PARITY " + json.dumps({
        "plan": name, "oracle_loss": loss, "oracle_bf16_points_loss": eloss, "torch_bf16_loss": tloss,
        "losses": [float(r["losses"][0]) for r in ranks],
        "worst": {"grad_vs_oracle": max(ours_g.values()), "torch_bf16_vs_oracle": max(floor.values()),
                  "grad_vs_bf16_points": max(emu_g.values()), "weight_vs_oracle": max(ours_w.values()),
                  "weight_vs_bf16_points": max(emu_w.values())},
        "per_tensor [grad_vs_oracle, torch_bf16_vs_oracle, grad_vs_bf16pts, w_vs_oracle, w_vs_bf16pts]":
            rows}))
    assert held == set(floor), set(floor) - held  # every tensor is held somewhere
    for r in ranks:
        assert abs(float(r["losses"][0]) - loss) <= RTOL * abs(loss), (r["losses"][0], loss)
    bad = {t: v for t, v in rows.items()
           if not (ours_g[t] <= 1.25 * floor[t] + 2e-3 and emu_g[t] <= max(RTOL, floor[t])
                   and ours_w[t] < RTOL and emu_w[t] < RTOL)}
    assert not bad, bad


def test_llama7b_shape_single_gpu():
    """Headline layer shape on one B200 vs the oracle."""
    if ngpu() < 1:
        pytest.skip("no CUDA device")
    res = run_inprocess("llama7b_2l_1gpu", steps=1)
    st = json.loads(bytes(res["stats"]).decode())
    assert st["launches_last_step"] > 0
    _check("llama7b_2l_1gpu", [res])


def test_llama7b_shape_tp31_two_gpus(tmp_path):
    if ngpu() < world_of("llama7b_2l_tp31"):
        pytest.skip("needs 2 GPUs")
    _check("llama7b_2l_tp31", run_plan("llama7b_2l_tp31", tmp_path, timeout=1200))


@pytest.mark.parametrize("name", ["llama13b_2l_1gpu", "llama30b_2l_1gpu"])
def test_large_layer_shapes_single_gpu(name):
    if ngpu() < 1:
        pytest.skip("no CUDA device")
    _check(name, [run_inprocess(name, steps=1)])


@pytest.mark.parametrize("name", ["llama13b_2l_tp31", "llama30b_2l_tp31"])
def test_large_layer_shapes_tp31(tmp_path, name):
    if ngpu() < world_of(name):
        pytest.skip("needs 2 GPUs")
    _check(name, run_plan(name, tmp_path, timeout=1200))


@pytest.mark.parametrize("name", ["llama13b_4l_pp3", "llama13b_4l_mixed", "llama13b_4l_tp3"])
def test_13b_four_gpu_plans(tmp_path, name):
    """cfg4 analogues at 13B layer shapes: 3-stage PP (uneven split, uneven
    TP stage); mixed TP + PP + DP with mismatched TP degrees; cfg4's uneven
    TP = 3 stage (widths 2:2:1 -> heads 16/16/8, two peers per exchange)."""
    if ngpu() < world_of(name):
        pytest.skip("needs 4 GPUs")
    ranks = run_plan(name, tmp_path, timeout=1200)
    _check(name, ranks)
    st = [json.loads(bytes(r["stats"]).decode()) for r in ranks]
    # the half-tier B200s run in green contexts with their SM share
    caps = {s["rank"]: (s["sm_cap_mode"], s["sm_applied"]) for s in st}
    assert caps[2][0] == "green" and caps[2][1] < caps[0][1], caps


@pytest.mark.parametrize("name", ["llama7b_2l_1gpu", "llama13b_2l_1gpu"])
def test_oracle_pinned_by_torch_fp32(name):
    """The numpy fp32 oracle vs an independent PyTorch fp32 autograd
    restatement of the same step (cuda:0, no TF32) at the benchmarked layer
    shapes: every gradient within 1e-4 normwise (the fp32 bar)."""
    if ngpu() < 1:
        pytest.skip("no CUDA device")
    import torch
    assert not torch.backends.cuda.matmul.allow_tf32
    loss, G, _ = oracle_for(name, keep=False)
    tloss, err = torch_floor(name, G, dtype="fp32")
    print("PIN " + json.dumps({"plan": name, "oracle_loss": loss, "torch_fp32_loss": tloss,
                               "worst": max(err.values())}))
    assert abs(tloss - loss) <= 1e-5 * abs(loss), (tloss, loss)
    assert max(err.values()) < 1e-4, err


@pytest.mark.parametrize("name", ["tiny_4_sched", "llama13b_4l_2_sched", "llama13b_4l_4_sched"])
def test_planner_plans_against_oracle(tmp_path, name):
    """Plans emitted by the reference's own scheduler / hierarchical graph
    partitioner (hexplan_schedule through oracle/_ref, committed by
    tests/golden/make_configs.py; scheduler.cpp:139-341, pipeline_layout.cpp:
    263-321): 4-stage PP of tiny on the [F, F, 1/2, 1/2] tiers; PP 3/1 of the
    13B layer shape on the capped pair; TP 2 + TP 2 stages (3/1 layers, two
    micro-batches of 2) on the tiers -- executed and checked like the hand
    plans."""
    if ngpu() < world_of(name):
        pytest.skip(f"needs {world_of(name)} GPUs")
    ranks = run_plan(name, tmp_path, timeout=1200)
    if name.startswith("tiny"):
        from parity_util import check_against_oracle
        check_against_oracle(name, ranks)
    else:
        _check(name, ranks)
