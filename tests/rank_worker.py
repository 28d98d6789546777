"""One executor rank for the multi-GPU parity tests (launched by
tests/test_executor_gpu.py with RANK / WORLD_SIZE / LOCAL_RANK / MASTER_*).

Runs `steps` training steps of configs/plans/<name>.json and saves, per rank,
the loss and every held tensor's reduced gradient and updated weights (after
the first step) to <out>/rank<r>.npz."""
import json
import re
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2409_01143_b200 import dist  # noqa: E402


def main():
    name, out = sys.argv[1], sys.argv[2]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    xcfg = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
    host_tokens = bool(int(sys.argv[5])) if len(sys.argv) > 5 else True
    idx = json.load(open(os.path.join(ROOT, "configs", "index.json")))[name]
    c = open(os.path.join(ROOT, "configs", "clusters", idx["cluster"] + ".json")).read()
    m = open(os.path.join(ROOT, "configs", "models", idx["model"] + ".json")).read()
    p = open(os.path.join(ROOT, "configs", "plans", name + ".json")).read()
    rank, world, local = dist.env_rank()
    ex = dist.make_executor(c, m, p, xcfg)
    res = {}
    losses = []
    for s in range(steps):
        tok = ex.synth_tokens(s) if (host_tokens and ex.role["active"]) else None
        losses.append(ex.step(tok))
        if s == 0 and ex.role["active"]:
            only = os.environ.get("HEXEXEC_TEST_READ")  # regex: read only these tensors
            for t in ex.role["tensors"]:
                if only and not re.search(only, t["name"]):
                    continue
                res[t["name"] + "|grad"] = ex.read(t["name"], 1)
                res[t["name"] + "|w"] = ex.read(t["name"], 0)
                res[t["name"] + "|row0"] = np.int64(t["row0"])
    if os.environ.get("HEXEXEC_TEST_SMPROBE") and ex.role["active"]:
        # SM placement of this rank's work after the steps (graph replays done)
        n = 4 * 148
        res["smid_stream"] = ex.sm_probe(0, n)
        res["smid_comm"] = ex.sm_probe(1, n)
        res["smid_gemm"] = ex.sm_probe(2, n)
    res["losses"] = np.array(losses, np.float64)
    res["stats"] = np.frombuffer(json.dumps(ex.stats()).encode(), np.uint8)
    np.savez(os.path.join(out, f"rank{rank}.npz"), **res)
    ex.close()


if __name__ == "__main__":
    main()
