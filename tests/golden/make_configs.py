"""Writes the cluster / model / plan documents of the BASELINE configs.

Cluster and model documents follow the reference formats
(/root/reference/proj/src/json_io.cpp:80-191) plus extension keys the
reference parser ignores.  Planner plans (cfg3, cfg5, even-split baselines)
are produced by the reference scheduler itself (oracle/_ref, built by
oracle/Makefile) and committed under configs/ as fixtures, so nothing here
runs on the GPU box (test infrastructure: it is the only generator that
links the compiled reference).

    python tests/golden/make_configs.py     # needs oracle/_ref/libhexplan_ref.so
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HERE = os.path.join(ROOT, "configs")
sys.path.insert(0, ROOT)

F, HALF, THIRD = 2250.0, 1125.0, 750.0
# Closed-loop calibration: effective speeds of the SM-capped
# tiers measured on B200 (bench.py reference_cost_model.calibrated, r01:
# llama7b_4l_4_asym -> F 1258 / 1278, H 910 / 909; llama7b_4l_2_asym -> F 1271,
# T 525).  Power capping makes a capped B200 faster per SM than a full one
# (SM clocks 1940-1965 vs ~1450 MHz), so the tiers are not 1 : 1/2 : 1/3.
F_CAL, HALF_CAL, THIRD_CAL = 1270.0, 909.0, 525.0


def cluster(devs, machines=None, sm=None):
    """devs: [(id, peak_tflops)]; sm: {id: sm_fraction} pins the SM cap (the
    calibrated documents keep the nominal tiers' caps, SURVEY 8(b) extension)"""
    machines = machines or {"box": [d for d, _ in devs]}
    mdoc = {m: {"intra_bandwidth_gbps": 900, "intra_latency_us": 3} for m in machines}
    where = {d: m for m, ds in machines.items() for d in ds}
    out = {"machines": mdoc,
           "devices": [{"id": d, "machine": where[d], "memory_gib": 178, "peak_tflops": p}
                       for d, p in devs],
           "inter": {"bandwidth_gbps": 900, "latency_us": 3}}
    for d in out["devices"]:
        if sm and d["id"] in sm:
            d["sm_fraction"] = sm[d["id"]]
    return out


TIERS8 = [("g0", F), ("g1", F), ("g2", F), ("g3", F), ("g4", HALF), ("g5", HALF),
          ("g6", THIRD), ("g7", THIRD)]
CLUSTERS = {
    "b200_1": cluster([("g0", F)]),
    "b200_2_capped": cluster([("g0", F), ("g1", THIRD)]),
    "b200_2_even": cluster([("g0", F), ("g1", F)]),
    "b200_4_tiers": cluster([("g0", F), ("g1", F), ("g2", HALF), ("g3", HALF)]),
    "b200_4_even": cluster([("g0", F), ("g1", F), ("g2", F), ("g3", F)]),
    "b200_8_onebox": cluster(TIERS8),
    "b200_8_tiers": cluster(TIERS8, {"tierF": ["g0", "g1", "g2", "g3"], "tierH": ["g4", "g5"],
                                     "tierT": ["g6", "g7"]}),
    "b200_8_even": cluster([(f"g{i}", F) for i in range(8)]),
    "b200_4_ht": cluster([("g0", HALF), ("g1", HALF), ("g2", THIRD), ("g3", THIRD)]),
    # homogeneous clusters with the SAME aggregate compute as the capped ones
    # (the "even-split plan at equal aggregate compute" comparison)
    "b200_2_eq": cluster([(f"g{i}", (F + THIRD) / 2) for i in range(2)]),
    "b200_4_eq": cluster([(f"g{i}", (2 * F + 2 * HALF) / 4) for i in range(4)]),
    "b200_8_eq": cluster([(f"g{i}", (4 * F + 2 * HALF + 2 * THIRD) / 8) for i in range(8)]),
    # calibrated tier speeds, same SM caps as the nominal tier clusters
    "b200_2_capped_cal": cluster([("g0", F_CAL), ("g1", THIRD_CAL)], sm={"g0": 1.0, "g1": 1 / 3}),
    "b200_4_tiers_cal": cluster([("g0", F_CAL), ("g1", F_CAL), ("g2", HALF_CAL), ("g3", HALF_CAL)],
                                sm={"g0": 1.0, "g1": 1.0, "g2": 0.5, "g3": 0.5}),
    "b200_8_onebox_cal": cluster(
        [("g0", F_CAL), ("g1", F_CAL), ("g2", F_CAL), ("g3", F_CAL), ("g4", HALF_CAL),
         ("g5", HALF_CAL), ("g6", THIRD_CAL), ("g7", THIRD_CAL)],
        sm={"g0": 1.0, "g1": 1.0, "g2": 1.0, "g3": 1.0, "g4": 0.5, "g5": 0.5, "g6": 1 / 3,
            "g7": 1 / 3}),
}

MODELS = {
    "tiny": {"num_layers": 4, "hidden_dim": 256, "seq_len": 128, "bytes_per_element": 4,
             "num_heads": 4, "ffn_dim": 1024, "vocab_size": 512},
    "llama7b_4l": {"num_layers": 4, "hidden_dim": 4096, "seq_len": 2048, "bytes_per_element": 2,
                   "num_heads": 32, "ffn_dim": 11008, "vocab_size": 32000},
    "llama7b": {"num_layers": 32, "hidden_dim": 4096, "seq_len": 2048, "bytes_per_element": 2,
                "num_heads": 32, "ffn_dim": 11008, "vocab_size": 32000},
    "llama13b": {"num_layers": 40, "hidden_dim": 5120, "seq_len": 2048, "bytes_per_element": 2,
                 "num_heads": 40, "ffn_dim": 13824, "vocab_size": 32000},
    "llama30b": {"num_layers": 60, "hidden_dim": 6656, "seq_len": 2048, "bytes_per_element": 2,
                 "num_heads": 52, "ffn_dim": 17920, "vocab_size": 32000},
    # 2-layer, short-sequence cuts of the 13B / 30B layer shapes (GPU sharding-
    # invariance tests of the H = 5120 / 6656, 40 / 52-head, F = 13824 / 17920 paths)
    "llama13b_2l_s256": {"num_layers": 2, "hidden_dim": 5120, "seq_len": 256,
                         "bytes_per_element": 2, "num_heads": 40, "ffn_dim": 13824,
                         "vocab_size": 1024},
    "llama30b_2l_s256": {"num_layers": 2, "hidden_dim": 6656, "seq_len": 256,
                         "bytes_per_element": 2, "num_heads": 52, "ffn_dim": 17920,
                         "vocab_size": 1024},
    # head_dim 256 (beyond the fused attention kernels' 64 / 128): the executor
    # runs the unfused GEMM + softmax attention
    "tiny_d256": {"num_layers": 2, "hidden_dim": 512, "seq_len": 128, "bytes_per_element": 4,
                  "num_heads": 2, "ffn_dim": 1024, "vocab_size": 512},
    # the benchmarked 7B shape (H 4096, 32 heads, F 11008, V 32000, S 2048) cut
    # to 2 layers: GPU-vs-oracle parity of the headline workload's kernels
    "llama7b_2l": {"num_layers": 2, "hidden_dim": 4096, "seq_len": 2048, "bytes_per_element": 2,
                   "num_heads": 32, "ffn_dim": 11008, "vocab_size": 32000},
    # 13B layer shapes, 4 layers: the 4-GPU analogues of cfg4 (3-stage PP with an
    # uneven TP stage) and of a mixed TP + PP + DP plan, against the oracle
    "llama13b_4l_s256": {"num_layers": 4, "hidden_dim": 5120, "seq_len": 256,
                         "bytes_per_element": 2, "num_heads": 40, "ffn_dim": 13824,
                         "vocab_size": 1024},
}


def stage(devs, start, count, widths=None):
    s = {"devices": devs, "tp": len(devs), "layer_start": start, "layer_count": count}
    if widths:
        s["tp_widths"] = widths
    return s


def pipe(batch, mb, stages):
    return {"batch": batch, "micro_batch": mb, "num_micro_batches": batch // mb,
            "stages": stages}


def plan(pipes, L):
    gb = sum(p["batch"] for p in pipes)
    groups = [{"layer": l, "members": []} for l in range(L)]
    for p in pipes:
        for s in p["stages"]:
            for l in range(s["layer_start"], s["layer_start"] + s["layer_count"]):
                groups[l]["members"].append(s["devices"][0])
    return {"global_batch": gb, "pipelines": pipes, "dp_groups": groups}


HAND = {
    # cfg1: tiny GPT, 2-rank asymmetric plans (TP widths 3:1; DP micro-batches 5:3)
    "tiny_1": ("b200_1", "tiny", plan([pipe(8, 4, [stage(["g0"], 0, 4)])], 4)),
    "tiny_tp31": ("b200_2_capped", "tiny", plan([pipe(8, 4, [stage(["g0", "g1"], 0, 4, [3, 1])])], 4)),
    "tiny_dp53": ("b200_2_capped", "tiny", plan([pipe(5, 1, [stage(["g0"], 0, 4)]),
                                                 pipe(3, 1, [stage(["g1"], 0, 4)])], 4)),
    "tiny_pp31": ("b200_2_capped", "tiny", plan([pipe(8, 2, [stage(["g0"], 0, 3),
                                                             stage(["g1"], 3, 1)])], 4)),
    "tiny_mixed4": ("b200_4_tiers", "tiny", plan([
        pipe(5, 1, [stage(["g0", "g2"], 0, 3, [2, 1]), stage(["g3"], 3, 1)]),
        pipe(3, 1, [stage(["g1"], 0, 4)])], 4)),
    "tiny_pp3_4": ("b200_4_tiers", "tiny", plan([pipe(8, 2, [
        stage(["g0"], 0, 2), stage(["g2", "g3"], 2, 1, [1, 3]), stage(["g1"], 3, 1)])], 4)),
    # same pipeline, middle stage listed out of rank order ([g3, g2], widths 3:1):
    # its TP communicator's rank 0 (lowest world rank) is not the stage leader
    "tiny_pp3_4_perm": ("b200_4_tiers", "tiny", plan([pipe(8, 2, [
        stage(["g0"], 0, 2), stage(["g3", "g2"], 2, 1, [3, 1]), stage(["g1"], 3, 1)])], 4)),
    "tiny_d256_1": ("b200_1", "tiny_d256", plan([pipe(4, 2, [stage(["g0"], 0, 2)])], 2)),
    # one micro-batch of 160 x 128 = 20480 tokens (> 16384: the embedding
    # backward sorts 64-bit keys with the device radix sort)
    "tiny_bigmb": ("b200_1", "tiny", plan([pipe(160, 160, [stage(["g0"], 0, 4)])], 4)),
    # N=1 workload: the cfg2 model on one B200
    "llama7b_4l_1gpu": ("b200_1", "llama7b_4l", plan([pipe(8, 1, [stage(["g0"], 0, 4)])], 4)),
    # cfg2: Llama-7B 4-layer block, TP=2 with 3:1 widths, rank 1 capped to 1/3 SMs
    "llama7b_4l_tp31": ("b200_2_capped", "llama7b_4l",
                        plan([pipe(8, 1, [stage(["g0", "g1"], 0, 4, [3, 1])])], 4)),
    "llama7b_4l_tp11_even": ("b200_2_even", "llama7b_4l",
                             plan([pipe(8, 1, [stage(["g0", "g1"], 0, 4)])], 4)),
    # the equivalent even-split of cfg2: TP=2 with equal widths on two
    # homogeneous devices of the same aggregate compute
    "llama7b_4l_tp11_eq": ("b200_2_eq", "llama7b_4l",
                           plan([pipe(8, 1, [stage(["g0", "g1"], 0, 4)])], 4)),
    # 4-GPU analogue of the calibrated 8-GPU plan's structure at full 7B size:
    # PP 16/16 on the F pair, TP=2 over the H pair, DP across mismatched TP
    "llama7b_4_mix": ("b200_4_tiers_cal", "llama7b", plan([
        pipe(20, 1, [stage(["g0"], 0, 16), stage(["g1"], 16, 16)]),
        pipe(12, 1, [stage(["g2", "g3"], 0, 32)])], 32)),
    "llama13b_2l_1gpu": ("b200_1", "llama13b_2l_s256", plan([pipe(2, 1, [stage(["g0"], 0, 2)])], 2)),
    "llama13b_2l_tp31": ("b200_2_capped", "llama13b_2l_s256",
                         plan([pipe(2, 1, [stage(["g0", "g1"], 0, 2, [3, 1])])], 2)),
    "llama30b_2l_1gpu": ("b200_1", "llama30b_2l_s256", plan([pipe(2, 1, [stage(["g0"], 0, 2)])], 2)),
    "llama30b_2l_tp31": ("b200_2_capped", "llama30b_2l_s256",
                         plan([pipe(2, 1, [stage(["g0", "g1"], 0, 2, [3, 1])])], 2)),
    # oracle parity at the benchmarked 7B shape: one B200, and TP 3:1 on the
    # capped pair (shards 24/8 heads, 8256/2752 FFN columns, 24000/8000 vocab rows)
    "llama7b_2l_1gpu": ("b200_1", "llama7b_2l", plan([pipe(2, 1, [stage(["g0"], 0, 2)])], 2)),
    "llama7b_2l_tp31": ("b200_2_capped", "llama7b_2l",
                        plan([pipe(2, 1, [stage(["g0", "g1"], 0, 2, [3, 1])])], 2)),
    # cfg4 analogue on 4 GPUs at 13B layer shapes: 3 stages with an uneven layer
    # split 2/1/1 and an uneven TP stage (3:1 over a full and a half-capped B200)
    "llama13b_4l_pp3": ("b200_4_tiers", "llama13b_4l_s256", plan([pipe(4, 1, [
        stage(["g0"], 0, 2), stage(["g1", "g2"], 2, 1, [3, 1]), stage(["g3"], 3, 1)])], 4)),
    # cfg4's uneven TP=3 stage (widths 2:2:1, as llama13b_pp3_asymtp) at 13B
    # layer shapes: TP 3 over [F, F, 1/2] for layers 0-2, then one 1/2 B200
    "llama13b_4l_tp3": ("b200_4_tiers", "llama13b_4l_s256", plan([pipe(4, 1, [
        stage(["g0", "g1", "g2"], 0, 3, [2, 2, 1]), stage(["g3"], 3, 1)])], 4)),
    # mixed TP + PP + DP at 13B layer shapes: pipeline 0 = TP 2:1 stage (3 layers)
    # + 1-layer stage, 3 samples; pipeline 1 = one B200, 2 samples
    "llama13b_4l_mixed": ("b200_4_tiers", "llama13b_4l_s256", plan([
        pipe(3, 1, [stage(["g0", "g2"], 0, 3, [2, 1]), stage(["g3"], 3, 1)]),
        pipe(2, 1, [stage(["g1"], 0, 4)])], 4)),
    # the pipelines of the calibrated 8-GPU plan (llama7b_8_cal) run alone:
    # P0 / P1 = PP 16/16 on two full B200s (21 samples); P2 = TP 2 on the half
    # tier (20 layers) + TP 2 on the third tier (12 layers), 22 samples
    "llama7b_cal_p0": ("b200_2_even", "llama7b", plan([
        pipe(21, 1, [stage(["g0"], 0, 16), stage(["g1"], 16, 16)])], 32)),
    "llama7b_cal_p2": ("b200_4_ht", "llama7b", plan([
        pipe(22, 1, [stage(["g0", "g1"], 0, 20), stage(["g2", "g3"], 20, 12)])], 32)),
    # cfg2 with widths from the calibrated speeds (1270 : 525 ~ 5 : 2)
    "llama7b_4l_tp52": ("b200_2_capped", "llama7b_4l",
                        plan([pipe(8, 1, [stage(["g0", "g1"], 0, 4, [5, 2])])], 4)),
    # width sweep of cfg2 around the delivered-compute ratio (148 SMs x 1.54 GHz :
    # 56 SMs x 1.97 GHz ~ 2.1 : 1)
    "llama7b_4l_tp73": ("b200_2_capped", "llama7b_4l",
                        plan([pipe(8, 1, [stage(["g0", "g1"], 0, 4, [7, 3])])], 4)),
    "llama7b_4l_tp21": ("b200_2_capped", "llama7b_4l",
                        plan([pipe(8, 1, [stage(["g0", "g1"], 0, 4, [2, 1])])], 4)),
    # cfg4: Llama-13B, 3 stages 16/14/10, asymmetric TP inside stages
    "llama13b_pp3_asymtp": ("b200_8_onebox", "llama13b", plan([pipe(16, 1, [
        stage(["g0", "g1", "g4"], 0, 16, [2, 2, 1]),
        stage(["g2", "g3", "g5"], 16, 14, [2, 2, 1]),
        stage(["g6", "g7"], 30, 10)])], 40)),
}

PLANNED = {
    # planner-emitted plans small enough for oracle parity on 2 / 4 GPUs (the
    # hierarchical partitioner + scheduler choose the PP / TP / micro-batch shape)
    "tiny_4_sched": ("b200_4_tiers", "tiny", "schedule",
                     {"global_batch": 8, "iterations": 30, "seed": 0, "threads": 8,
                      "state_multiplier": 2.5}),
    "llama13b_4l_2_sched": ("b200_2_capped", "llama13b_4l_s256", "schedule",
                            {"global_batch": 6, "iterations": 30, "seed": 0, "threads": 8,
                             "state_multiplier": 2.5}),
    "llama13b_4l_4_sched": ("b200_4_tiers", "llama13b_4l_s256", "schedule",
                            {"global_batch": 8, "iterations": 30, "seed": 0, "threads": 8,
                             "state_multiplier": 2.5}),
    # cfg3: Llama-7B on 8 B200 tiers; asymmetric DP with uneven micro-batch counts
    "llama7b_8_asym": ("b200_8_onebox", "llama7b", "schedule",
                       {"global_batch": 64, "iterations": 50, "seed": 0, "threads": 8,
                        "state_multiplier": 2.5}),
    "llama7b_8_even": ("b200_8_even", "llama7b", "symmetric",
                       {"global_batch": 64, "iterations": 50, "seed": 0, "threads": 8,
                        "state_multiplier": 2.5}),
    # cfg5: Llama-30B layers under a full plan from the hierarchical partitioner
    "llama30b_8_tiers": ("b200_8_tiers", "llama30b", "schedule",
                         {"global_batch": 64, "iterations": 50, "seed": 0, "threads": 8,
                          "state_multiplier": 2.5}),
    # N=4 scaling point
    "llama7b_4l_4_asym": ("b200_4_tiers", "llama7b_4l", "schedule",
                          {"global_batch": 48, "iterations": 30, "seed": 0, "threads": 8,
                           "state_multiplier": 2.5}),
    "llama7b_4l_2_asym": ("b200_2_capped", "llama7b_4l", "schedule",
                          {"global_batch": 8, "iterations": 20, "seed": 0, "threads": 8,
                           "state_multiplier": 2.5}),
    # the reference scheduler on the calibrated tier speeds
    "llama7b_4l_2_cal": ("b200_2_capped_cal", "llama7b_4l", "schedule",
                         {"global_batch": 8, "iterations": 20, "seed": 0, "threads": 8,
                          "state_multiplier": 2.5}),
    "llama7b_4l_4_cal": ("b200_4_tiers_cal", "llama7b_4l", "schedule",
                         {"global_batch": 48, "iterations": 30, "seed": 0, "threads": 8,
                          "state_multiplier": 2.5}),
    "llama7b_8_cal": ("b200_8_onebox_cal", "llama7b", "schedule",
                      {"global_batch": 64, "iterations": 50, "seed": 0, "threads": 8,
                       "state_multiplier": 2.5}),
    # even-split plans (hexplan_symmetric_baseline) at equal aggregate compute
    "llama7b_4l_2_even": ("b200_2_eq", "llama7b_4l", "symmetric",
                          {"global_batch": 8, "iterations": 20, "seed": 0, "threads": 8,
                           "state_multiplier": 2.5}),
    "llama7b_4l_4_even": ("b200_4_eq", "llama7b_4l", "symmetric",
                          {"global_batch": 48, "iterations": 30, "seed": 0, "threads": 8,
                           "state_multiplier": 2.5}),
    "llama7b_8_eq_even": ("b200_8_eq", "llama7b", "symmetric",
                          {"global_batch": 64, "iterations": 50, "seed": 0, "threads": 8,
                           "state_multiplier": 2.5}),
}


def write(path, obj):
    with open(path, "w") as f:
        json.dump(obj, f, indent=2)
        f.write("\n")


def main():
    for sub in ("clusters", "models", "plans"):
        os.makedirs(os.path.join(HERE, sub), exist_ok=True)
    for k, v in CLUSTERS.items():
        write(os.path.join(HERE, "clusters", k + ".json"), v)
    for k, v in MODELS.items():
        write(os.path.join(HERE, "models", k + ".json"), v)
    index = {}
    for k, (c, m, p) in HAND.items():
        write(os.path.join(HERE, "plans", k + ".json"), p)
        index[k] = {"cluster": c, "model": m, "source": "hand"}
    from oracle import refshim
    for k, (c, m, kind, cfg) in PLANNED.items():
        res = refshim.plan(json.dumps(CLUSTERS[c]), json.dumps(MODELS[m]), json.dumps(cfg), kind)
        assert res["found"], (k, res)
        with open(os.path.join(HERE, "plans", k + ".json"), "w") as f:
            f.write(res["plan"])
        index[k] = {"cluster": c, "model": m, "source": f"hexplan_{kind}", "config": cfg,
                    "predicted_s": res["cost"], "predicted_mfu": res["mfu"]}
        print(k, round(res["cost"], 6), round(res["mfu"], 4))
    write(os.path.join(HERE, "index.json"), index)


if __name__ == "__main__":
    main()
