"""Where the bf16 executor lands against the fp32 oracle, next to PyTorch's
own bf16 autocast step on the same weights / tokens (tests/torch_bf16_ref.py).

    python scripts/bf16_floor.py llama13b_2l_1gpu [llama7b_2l_1gpu ...] [--variants]

Prints one JSON line per plan: per-tensor normwise relative gradient error of
(a) the executor vs the oracle, (b) torch bf16 vs the oracle, (c) torch fp32
vs the oracle (sanity), (d) the executor vs torch bf16."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def main():
    from oracle import numeric as O
    from paper_2409_01143_b200 import Executor
    import torch_bf16_ref as TR
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    variants = [{}]
    if "--variants" in sys.argv:
        variants += [{"attention": "unfused"}, {"fuse_rope": False, "fuse_swiglu": False}]
    idx = json.load(open(os.path.join(ROOT, "configs", "index.json")))
    for name in names:
        e = idx[name]
        c = open(os.path.join(ROOT, "configs", "clusters", e["cluster"] + ".json")).read()
        m = open(os.path.join(ROOT, "configs", "models", e["model"] + ".json")).read()
        p = open(os.path.join(ROOT, "configs", "plans", name + ".json")).read()
        st = O.Step(json.loads(c), json.loads(m), p)
        loss_o, G, _ = st.run(0)
        stb = O.Step(json.loads(c), json.loads(m), p, bf16_points=True)
        loss_e, Ge, _ = stb.run(0)
        del stb
        st2 = O.Step(json.loads(c), json.loads(m), p)  # fresh initial weights
        loss_b, Gb = TR.step_grads(st2, dtype="bf16")
        loss_f, Gf = TR.step_grads(st2, dtype="fp32")
        out = {"plan": name, "oracle_loss": loss_o, "oracle_bf16_points_loss": loss_e,
               "torch_bf16_loss": loss_b,
               "torch_fp32_loss": loss_f, "variants": []}
        for xc in variants:
            ex = Executor(c, m, p, xc, rank=0, world_size=1, device=0)
            loss = ex.step(ex.synth_tokens(0))
            rows = {}
            for t in ex.role["tensors"]:
                g = ex.read(t["name"], 1)
                n = t["name"]
                rows[n] = [round(rel(g, G[n]), 5), round(rel(Gb[n], G[n]), 5),
                           round(rel(Gf[n], G[n]), 7), round(rel(g, Gb[n]), 5),
                           round(rel(g, Ge[n]), 5), round(rel(Ge[n], G[n]), 5)]
            ex.close()
            worst = {k: max(v[i] for v in rows.values()) for i, k in
                     enumerate(["ours_vs_oracle", "torch_bf16_vs_oracle", "torch_fp32_vs_oracle",
                                "ours_vs_torch_bf16", "ours_vs_oracle_bf16_points",
                                "oracle_bf16_points_vs_oracle"])}
            out["variants"].append({"exec_config": xc, "loss": loss, "worst": worst,
                                    "per_tensor [ours, torch_bf16, torch_fp32, ours_vs_torch, ours_vs_bf16pts, bf16pts]": rows})
        print("BF16FLOOR " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
