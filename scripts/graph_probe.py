"""Multi-rank CUDA-graph probe mirroring bench.py's call sequence (debug aid)."""
import faulthandler
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_01143_b200 import dist  # noqa: E402


def main():
    faulthandler.dump_traceback_later(60, exit=True)
    name, xcfg, seq = sys.argv[1], json.loads(sys.argv[2]), sys.argv[3]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    idx = json.load(open(os.path.join(root, "configs", "index.json")))[name]
    c = open(os.path.join(root, "configs", "clusters", idx["cluster"] + ".json")).read()
    m = open(os.path.join(root, "configs", "models", idx["model"] + ".json")).read()
    p = open(os.path.join(root, "configs", "plans", name + ".json")).read()
    rank, world, _ = dist.env_rank()
    ex = dist.make_executor(c, m, p, xcfg, tag=f"uid-{name}")
    t0 = time.time()
    for i, op in enumerate(seq):
        if op == "p":
            ex.set_profile(True)
        elif op == "q":
            ex.set_profile(False)
        elif op == "a":
            ex.step_async()
        elif op == "s":
            ex.sync()
        elif op == "h":
            ex.step(ex.synth_tokens(100 + i) if ex.role["active"] else None)
        elif op == "d":
            ex.step(None)
        elif op == "b":
            dist.barrier(rank, world, f"b{i}")
        print(f"rank {rank} op {i}:{op} ok", flush=True)
    ex.sync()
    print(f"rank {rank} done {time.time() - t0:.2f}s loss {ex.last_loss():.4f}", flush=True)
    ex.close()
    print(f"rank {rank} closed", flush=True)


if __name__ == "__main__":
    main()
