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
