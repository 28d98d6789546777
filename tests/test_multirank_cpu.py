"""Host side of the N > 1 path on CPU (no GPU): world-size 2 and 4 process
groups over gloo, one process per rank like torchrun.  Each rank exchanges
the NCCL unique id through the TCPStore (paper_2409_01143_b200/dist.py),
creates its validate_only executor (layout + memory sizing) for multi-rank
plans, and the ranks check with gloo collectives that they derived the same
layout, that every chunk-matched DP communicator sees the same bucket
sequence on all its members (the grouped ncclAllReduce calls must match
call for call), and that the PP send / receive peers pair up; the bench's
max-over-ranks reduction runs over the same store."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,plans", [
    (2, "tiny_tp31,tiny_dp53,tiny_pp31,llama7b_4l_tp31,llama7b_2l_tp31,llama13b_2l_tp31"),
    (4, "tiny_mixed4,tiny_pp3_4,tiny_pp3_4_perm,llama13b_4l_pp3,llama13b_4l_mixed,llama13b_4l_tp3,"
        "llama7b_4l_4_cal,llama7b_4l_4_even"),
])
def test_multirank_host_path_gloo(world, plans):
    pytest.importorskip("torch.distributed")
    for attempt in range(3):
        port = _port()
        procs = []
        for r in range(world):
            env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                       MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
            procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mr_worker.py"),
                                           plans], env=env, stdout=subprocess.PIPE,
                                          stderr=subprocess.PIPE, text=True))
        outs = [p.communicate(timeout=300) for p in procs]
        if all(p.returncode == 0 for p in procs):
            break
        if not any("EADDRINUSE" in e or "address already in use" in e.lower() for _, e in outs):
            break
    assert all(p.returncode == 0 for p in procs), [e[-2000:] for _, e in outs]
    res = [json.loads([l for l in o.splitlines() if l.startswith("MR ")][-1][3:]) for o, _ in outs]
    for r in res:
        assert r.get("uid_same", True), r
        n = 0
        for name in plans.split(","):
            if name not in r:
                continue
            n += 1
            v = r[name]
            assert v["layout_same"] and v["bucket_seq_agree"] and v["pp_symmetric"], (name, v)
            assert v["arena_max"] >= v["arena_bytes"] > 0 or not v["active"], (name, v)
        assert n >= 3
