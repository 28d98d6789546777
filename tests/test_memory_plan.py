"""Host-only dry run of every BASELINE plan: each rank's HBM arena (weights,
fp32 master + AdamW state, grads, DP comm buffer, 1F1B activation slots,
scratch) must fit a B200 (183 GB; 8 GiB kept for the CUDA context, NCCL and
the TMEM-less runtime).  Exercises hexexec_ctx_create(validate_only)."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = os.path.join(ROOT, "configs")
INDEX = json.load(open(os.path.join(CFG, "index.json")))
B200_BYTES = 183359 * 2**20
HEADROOM = 8 * 2**30


@pytest.mark.parametrize("name", sorted(INDEX))
def test_every_rank_fits(name):
    from paper_2409_01143_b200.hexexec import Executor
    e = INDEX[name]
    c = open(os.path.join(CFG, "clusters", e["cluster"] + ".json")).read()
    m = open(os.path.join(CFG, "models", e["model"] + ".json")).read()
    p = open(os.path.join(CFG, "plans", name + ".json")).read()
    world = len(json.loads(c)["devices"])
    worst = 0
    for r in range(world):
        ex = Executor(c, m, p, {"validate_only": True}, rank=r, world_size=world)
        st = ex.stats()
        worst = max(worst, st["arena_bytes"])
        ex.close()
    assert worst + HEADROOM <= B200_BYTES, (name, worst / 2**30)


def _dry(c, m, p, cfg, world):
    from paper_2409_01143_b200.hexexec import Executor
    worst = 0
    for r in range(world):
        ex = Executor(c, m, p, dict(cfg, validate_only=True), rank=r, world_size=world)
        worst = max(worst, ex.stats()["arena_bytes"])
        ex.close()
    return worst


def test_recompute_shrinks_activation_memory_and_memory_gib_caps():
    """Activation recompute keeps only layer inputs per 1F1B slot; the device's
    memory_gib (cost_model.cpp:130-153 mem_check) caps each rank's arena, so a
    memory tier that cannot hold stored activations runs with recompute."""
    from paper_2409_01143_b200.hexexec import HexexecError
    name = "llama13b_pp3_asymtp"
    e = INDEX[name]
    c = json.load(open(os.path.join(CFG, "clusters", e["cluster"] + ".json")))
    m = open(os.path.join(CFG, "models", e["model"] + ".json")).read()
    p = open(os.path.join(CFG, "plans", name + ".json")).read()
    world = len(c["devices"])
    # stored activations without weight-gradient grouping (auto grouping only
    # takes memory that is left over, so it never makes a plan infeasible)
    full = _dry(json.dumps(c), m, p, {"wgrad_group": 1}, world)
    rc = _dry(json.dumps(c), m, p, {"recompute": True}, world)
    assert rc < 0.9 * full, (rc / 2**30, full / 2**30)
    cap_gib = (rc + full) / 2 / 2**30
    for d in c["devices"]:
        d["memory_gib"] = cap_gib
    with pytest.raises(HexexecError) as ei:
        _dry(json.dumps(c), m, p, {"wgrad_group": 1}, world)
    assert "memory_gib" in str(ei.value)
    with pytest.raises(HexexecError):
        _dry(json.dumps(c), m, p, {"wgrad_group": -1}, world)
    assert _dry(json.dumps(c), m, p, {"recompute": True}, world) == rc
