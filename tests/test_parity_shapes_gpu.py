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

Large-shape oracles are not cached (several GB per copy); a summary of the
worst errors per tensor is printed (pytest -s) for the logs in profiles/.
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity_util import (RTOL, check_against_oracle, ngpu, oracle_for, rel,  # noqa: E402
                         run_inprocess, run_plan, world_of)


def _summary(name, ranks, report, oracle_loss):
    worst_g = max(report.items(), key=lambda kv: kv[1][0])
    worst_w = max(report.items(), key=lambda kv: kv[1][1])
    out = {"plan": name, "oracle_loss": oracle_loss,
           "losses": [float(r["losses"][0]) for r in ranks],
           "tensors": len(report),
           "worst_grad": [worst_g[0], worst_g[1][0]], "worst_weight": [worst_w[0], worst_w[1][1]]}
    print("PARITY " + json.dumps(out))


def _check(name, ranks):
    ora = oracle_for(name, keep=False)
    report = {}
    try:
        check_against_oracle(name, ranks, oracle=ora, report=report)
    finally:
        print("PARITY-ALL " + name + " " + json.dumps(
            {t: [round(a, 5), round(b, 5)] for t, (a, b) in sorted(report.items())}))
    _summary(name, ranks, report, ora[0])


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


@pytest.mark.parametrize("name", ["llama13b_4l_pp3", "llama13b_4l_mixed"])
def test_13b_four_gpu_plans(tmp_path, name):
    """cfg4 analogue (3-stage PP, uneven split, uneven TP stage) and mixed
    TP + PP + DP with mismatched TP degrees, at 13B layer shapes."""
    if ngpu() < world_of(name):
        pytest.skip("needs 4 GPUs")
    ranks = run_plan(name, tmp_path, timeout=1200)
    _check(name, ranks)
    st = [json.loads(bytes(r["stats"]).decode()) for r in ranks]
    # the half-tier B200s run in green contexts with their SM share
    caps = {s["rank"]: (s["sm_cap_mode"], s["sm_applied"]) for s in st}
    assert caps[2][0] == "green" and caps[2][1] < caps[0][1], caps
