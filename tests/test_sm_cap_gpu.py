"""SM caps of the emulated GPU tiers (PAPER.md:415-425 mixed-capability
clusters, emulated on homogeneous B200s; SURVEY §7 hard part (iv)).

On b200_2_capped the second device has peak_tflops 750 (sm_fraction 1/3 of
a 2250 TFLOPS B200): its rank must run in a CUDA green context holding
ceil(148/3) SMs rounded up to the driver's split granularity (56 on B200),
and every piece of its work must stay inside that partition:
  * probe CTAs on the executor stream and on the DP / comm stream,
  * a persistent tcgen05 GEMM (each CTA logs %smid),
while the uncapped rank spreads over the whole chip.  NCCL kernels are
launched on the same green-context streams (ncclAllReduce / ncclSend take the
executor's streams; the step graph captures them there), so the driver places
them in the same partition as the probe CTAs.
"""
import json
import math
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity_util import ngpu, run_plan  # noqa: E402


def test_sm_cap_green_context_partition(tmp_path):
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    ranks = run_plan("tiny_tp31", tmp_path, steps=2, env={"HEXEXEC_TEST_SMPROBE": "1"})
    st = [json.loads(bytes(r["stats"]).decode()) for r in ranks]
    total = st[0]["sm_total"]
    want = math.ceil(total / 3)
    # rank 0: full B200, no cap
    assert st[0]["sm_cap_mode"] == "none" and st[0]["sm_applied"] == total
    full = set(ranks[0]["smid_stream"].tolist())
    assert len(full) > total * 0.9, len(full)
    # rank 1: green context of >= ceil(148/3) SMs, rounded to the split granularity
    assert st[1]["sm_cap_mode"] == "green", st[1]
    applied = st[1]["sm_applied"]
    assert want <= applied < want + 16 and applied < total, (want, applied)
    if total == 148:
        assert applied == 56, applied  # B200: granularity 8 -> 49 rounds to 56
    part = set(ranks[1]["smid_stream"].tolist())
    comm = set(ranks[1]["smid_comm"].tolist())
    gemm = set(ranks[1]["smid_gemm"].tolist())
    assert len(part) <= applied and len(comm) <= applied, (len(part), len(comm), applied)
    assert comm <= part | comm and len(part | comm) <= applied, (sorted(part), sorted(comm))
    assert len(gemm) >= applied * 0.9 and gemm <= (part | comm), (len(gemm), sorted(gemm - part - comm))
    # the partition is actually used (the probe CTAs spread over it)
    assert len(part) >= applied * 0.9, (len(part), applied)
    print("SMCAP " + json.dumps({"rank1_applied": applied, "probe_sms": len(part),
                                 "comm_sms": len(comm), "gemm_sms": len(gemm),
                                 "rank0_probe_sms": len(full)}))
