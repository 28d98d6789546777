#!/usr/bin/env python
"""bench.py — tokens/s & MFU of one asymmetric-parallel training step executed
from a HexiScale plan on N B200s, vs the even-split plan at equal aggregate
compute, vs the CPU reference (BASELINE.json "metric").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--plan NAME] [--impl reference]

Launch for N > 1 (one rank per GPU):
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

A "step" = one full training step (fwd + bwd of every micro-batch, DP sync,
AdamW) of the plan over its global batch of synthetic tokens.  `value` is
device-timed (CUDA events on the executor stream, max over ranks) with the
tokens resident in HBM; `e2e` is the same step through the public C ABI
(hexexec_step) with host token buffers copied H2D and the loss read D2H
inside the timed region (host wall clock, max over ranks).
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
CFG = os.path.join(ROOT, "configs")

METRIC = "tokens/s & MFU per asym plan at 1/2/4/8 B200 vs even split + CPU ref"
# N -> (asymmetric plan, even-split plans at equal aggregate compute: the first
# keeps the asymmetric plan's parallel structure with even shares on a
# homogeneous cluster; the next is the reference's symmetric_baseline shape)
PLANS = {
    1: ("llama7b_4l_1gpu", None),
    2: ("llama7b_4l_tp31", "llama7b_4l_tp11_eq,llama7b_4l_2_even"),
    4: ("llama7b_4l_4_cal", "llama7b_4l_4_even"),
    8: ("llama7b_8_cal", "llama7b_8_eq_even"),
}
# further asymmetric arms reported beside the headline one: the nominal-tier
# planner plans (peak_tflops proportional to the SM share) and, for cfg2, the
# TP widths chosen from the calibrated speeds
ALT = {
    2: "llama7b_4l_tp52,llama7b_4l_2_cal",
    4: "llama7b_4l_4_asym",
    8: "llama7b_8_asym",
}
B200_SPEC = 2250.0


def peaks():
    p = {"bf16_tflops": 1661.7, "bf16_tflops_sustained": 1404.0, "hbm_gbs": 6553.0,
         "source": "fallback (MEASURED_PEAKS.json absent)"}
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        j = json.load(open(f))
        p.update({k: j[k] for k in ("bf16_tflops", "bf16_tflops_sustained", "hbm_gbs") if k in j})
        p["source"] = "MEASURED_PEAKS.json"
    return p


def load(name):
    idx = json.load(open(os.path.join(CFG, "index.json")))[name]
    c = open(os.path.join(CFG, "clusters", idx["cluster"] + ".json")).read()
    m = open(os.path.join(CFG, "models", idx["model"] + ".json")).read()
    p = open(os.path.join(CFG, "plans", name + ".json")).read()
    return c, m, p, idx


def full_model(c: str, m: str, p: str) -> dict:
    """The model document with the executor's defaults filled in (num_heads,
    ffn_dim, vocab_size, ...), from the product's own plan layout."""
    from paper_2409_01143_b200.hexexec import Plan
    pl = Plan(c, m, p)
    try:
        return pl.layout()["model"]
    finally:
        pl.close()


def model_flops(m: dict, tokens: int) -> tuple[float, float]:
    """(reference-convention FLOPs, exact causal Llama training FLOPs) for
    `tokens` trained tokens.  Reference: 72*S*H^2*(1+S/6H) per token per layer
    (cost_model.cpp:17-21, :260-265).  Exact: 3x forward GEMM flops incl. the
    causal attention products and the LM head."""
    L, H, S, F, V = m["num_layers"], m["hidden_dim"], m["seq_len"], m["ffn_dim"], m["vocab_size"]
    ref = 72.0 * S * H * H * (1 + S / (6.0 * H)) * L / S * tokens
    fwd = L * (2 * H * (4 * H + 3 * F) + 2 * S * H) + 2 * H * V
    return ref, 3.0 * fwd * tokens


class Clocks:
    """nvidia-smi sampler for the timed region (rank 0)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, n_gpus: int = 1):
        # the job's GPUs only (an idle GPU of the box would drag the median down)
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        ids = [x.strip() for x in vis.split(",")] if vis else [str(i) for i in range(n_gpus)]
        self.ids = ",".join(ids[:n_gpus])
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.t0 = self.t1 = None

    def start(self):
        """Start sampling (before the warm-up: nvidia-smi takes ~1 s to come up);
        only rows stamped inside [mark_begin, mark_end] are kept."""
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", self.ids, f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def mark_begin(self):
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        self.t1 = datetime.datetime.now()

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        per = {}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f")
                if self.t0 and self.t1 and not (self.t0 <= ts <= self.t1):
                    continue
                sm.append(float(r[2]))
                mx.append(float(r[3]))
                per.setdefault(r[1], []).append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for i, n in enumerate(names):
                if len(r) > 6 + i and r[6 + i].lower() == "active":
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "sm_mhz_per_gpu": {k: statistics.median(v) for k, v in sorted(per.items())},
                "gpu_of_rank": self.ids.split(","),
                "samples": len(sm)}


def gather_max(vals: list, rank: int, world: int, tag: str) -> list:
    """Max over ranks of a list of floats (TCPStore)."""
    if world == 1:
        return vals
    from paper_2409_01143_b200 import dist
    st = dist.store(rank, world)
    st.set(f"bench/{tag}/{rank}", json.dumps(vals))
    allv = [json.loads(st.get(f"bench/{tag}/{r}")) for r in range(world)]
    return [max(v[i] for v in allv) for i in range(len(vals))]


def gather_all(val, rank: int, world: int, tag: str) -> list:
    """Every rank's JSON value, in rank order (TCPStore)."""
    if world == 1:
        return [val]
    from paper_2409_01143_b200 import dist
    st = dist.store(rank, world)
    st.set(f"bench/{tag}/{rank}", json.dumps(val))
    return [json.loads(st.get(f"bench/{tag}/{r}")) for r in range(world)]


def gather_sum(vals: list, rank: int, world: int, tag: str) -> list:
    if world == 1:
        return vals
    from paper_2409_01143_b200 import dist
    st = dist.store(rank, world)
    st.set(f"bench/{tag}/{rank}", json.dumps(vals))
    allv = [json.loads(st.get(f"bench/{tag}/{r}")) for r in range(world)]
    return [sum(v[i] for v in allv) for i in range(len(vals))]


EXEC_CFG = {}  # --exec-config: extra executor config keys (e.g. {"recompute": true})
MAX_REF_LAYERS = 4  # layers of the CPU reference's bounded sample (the 4-layer workloads run whole)


def log(rank: int, msg: str):
    print(f"[bench rank {rank} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_plan(name: str, steps: int, warmup: int, rank: int, world: int, clocks: bool):
    from paper_2409_01143_b200 import dist
    c, m, p, idx = load(name)
    log(rank, f"{name}: creating executor")
    # per-GEMM CUDA events inside the step graph (one micro-batch per step):
    # the roofline is read from the timed replays themselves
    xc = {"graph_gemm_events": True}
    xc.update(EXEC_CFG)
    ex = dist.make_executor(c, m, p, xc, tag=f"uid-{name}")
    role = ex.role
    # ---- profiled pass first (eager, CUDA events around every GEMM and after every
    # op): roofline evidence for the TP GEMMs + per-kernel-class step timeline.
    # Eager NCCL work is kept before the first graph capture (no graph/eager mixing).
    log(rank, f"{name}: profiled pass")
    ex.set_profile(True)
    for _ in range(2):
        ex.step_async()
    ex.sync()
    st = ex.stats()
    ex.set_profile(False)
    # closed-loop calibration input: this rank's effective layer speed
    from paper_2409_01143_b200 import calibrate
    speeds = gather_all([role["device"], calibrate.device_speed(st, role, json.loads(m), 2),
                         st["sm_applied"] / max(st["sm_total"], 1)] if role["active"] else None,
                        rank, world, f"cal-{name}")
    ck = Clocks(world) if clocks else None
    if ck:
        ck.start()
    log(rank, f"{name}: warm-up {warmup}")
    for _ in range(warmup):      # first graph-mode step is captured into the CUDA graph
        ex.step_async()
    ex.sync()
    log(rank, f"{name}: timed {steps}")
    # ---- device-timed region (tokens resident in HBM)
    dist.barrier(rank, world, f"t0-{name}")
    if ck:
        ck.mark_begin()
    ex.timer_start()
    for _ in range(steps):
        ex.step_async()
    dev_ms = ex.timer_stop()
    if ck:
        ck.mark_end()
    clk = ck.stop() if ck else None
    ex.sync()  # reads the per-GEMM events of the last timed replay
    st_timed = ex.stats()
    launches_step = st_timed.get("launches_last_step", 0)
    dev_ms = gather_max([dev_ms], rank, world, f"dev-{name}")[0]
    # ---- e2e region: public API with host token buffers (H2D) + loss (D2H)
    log(rank, f"{name}: e2e {steps}")
    toks = [ex.synth_tokens(warmup + steps + s) if role["active"] else None for s in range(steps)]
    ck2 = Clocks(world) if clocks else None
    if ck2:
        ck2.start()
        time.sleep(1.0)  # nvidia-smi start-up
    dist.barrier(rank, world, f"e0-{name}")
    if ck2:
        ck2.mark_begin()
    t0 = time.perf_counter()
    loss = None
    for s in range(steps):
        loss = ex.step(toks[s])
    e2e_ms = (time.perf_counter() - t0) * 1e3
    if ck2:
        ck2.mark_end()
    clk_e2e = ck2.stop() if ck2 else None
    e2e_ms = gather_max([e2e_ms], rank, world, f"e2e-{name}")[0]
    # order check: the same device-timed loop once more after the e2e region
    # (e2e has come out 0.5-1 % above the device-timed value although it adds
    # copies and a host sync per step: a second device-timed pass shows how
    # much of that is position in the run rather than the measurement)
    dist.barrier(rank, world, f"t1-{name}")
    ex.timer_start()
    for _ in range(steps):
        ex.step_async()
    dev2_ms = gather_max([ex.timer_stop()], rank, world, f"dev2-{name}")[0]
    h2d = toks[0].nbytes if (role["active"] and toks[0] is not None) else 0
    gp = st.get("gemm_profile", {})
    lin = gp.get("tp_linear", {})
    sums = gather_sum([float(h2d), 4.0, float(launches_step),
                       float(lin.get("flops", 0.0)), float(lin.get("ms", 0.0)),
                       float(lin.get("launches", 0)),
                       float(st["sm_applied"]) / max(float(st["sm_total"]), 1.0)
                       if role["active"] else 0.0],
                      rank, world, f"sum-{name}")
    gg = st_timed.get("gemm_profile_graph")
    if gg:  # roofline from inside the timed region (events captured in the graph)
        lin = gg.get("tp_linear", {})
    share = float(st["sm_applied"]) / max(float(st["sm_total"]), 1.0) if role["active"] else 0.0
    tl_all = gather_all({k: round(v["ms"] / 2, 3) for k, v in st.get("timeline_ms", {}).items()},
                        rank, world, f"tl-{name}")
    tlg_all = gather_all({k: round(v["ms"], 4) for k, v in
                          st_timed.get("timeline_graph_one_mb", {}).items()}, rank, world,
                         f"tlg-{name}")
    per_rank = gather_all([float(lin.get("flops", 0.0)), float(lin.get("ms", 0.0)),
                           float(lin.get("launches", 0)), share], rank, world, f"lin-{name}")
    caps = gather_all({k: st.get(k) for k in ("rank", "active", "sm_cap_mode", "sm_applied",
                                              "sm_total", "sm_fraction")},
                      rank, world, f"cap-{name}")
    n_mb = gather_all(int(role.get("num_micro_batches", 0)) if role["active"] else 0, rank,
                      world, f"nmb-{name}")
    ex.close()
    log(rank, f"{name}: done")
    return dict(name=name, idx=idx, cluster=json.loads(c), model=json.loads(m),
                plan=json.loads(p), dev_ms=dev_ms, e2e_ms=e2e_ms, loss=loss, clocks=clk,
                clocks_e2e=clk_e2e, sm_caps=caps, n_mb=n_mb, dev2_ms=dev2_ms,
                stats=st, gemm_graph=gg, h2d=sums[0], d2h=sums[1], launches=sums[2], lin_flops=sums[3],
                lin_ms=sums[4], lin_launches=sums[5], sm_share=sums[6], lin_per_rank=per_rank, tl_all=tl_all, tlg_all=tlg_all,
                speeds=[x for x in speeds if x])


def summarize(r: dict, steps: int, pk: dict) -> dict:
    gb = r["plan"]["global_batch"]
    S = r["model"]["seq_len"]
    tokens = gb * S
    tps = tokens * steps / (r["dev_ms"] / 1e3)
    e2e = tokens * steps / (r["e2e_ms"] / 1e3)
    ref_f, exact_f = model_flops(full_model(json.dumps(r["cluster"]), json.dumps(r["model"]),
                                            json.dumps(r["plan"])), tokens)
    step_s = r["dev_ms"] / 1e3 / steps
    # aggregate peak of the emulated tiers: sum over ranks of applied SM share x measured peak
    agg = r["sm_share"] * pk["bf16_tflops"] * 1e12
    return {"plan": r["name"], "tokens_per_s": tps, "e2e_tokens_per_s": e2e,
            "ms_per_step": r["dev_ms"] / steps, "e2e_ms_per_step": r["e2e_ms"] / steps,
            "mfu_ref_convention": ref_f / step_s / agg if agg else None,
            "mfu_exact": exact_f / step_s / agg if agg else None,
            "aggregate_sm_share": r["sm_share"], "loss": r["loss"],
            "sm_ghz": sm_ghz(r), "tokens_per_s_per_sm_ghz": tps / sm_ghz(r) if sm_ghz(r) else None,
            # the same reference-convention FLOPs over the compute the ranks
            # actually delivered: sum_r SMs_r x median clock_r x 8192 dense bf16
            # FLOP / SM / clock (the B200 tensor rate: 2.25 PFLOP/s = 148 SMs x
            # 1.855 GHz x 8192); under the 1 kW cap a full-SM B200 clocks ~1.5-1.6
            # GHz while an SM-capped rank holds ~1.9-1.97 GHz
            "mfu_at_delivered_clock": (ref_f / step_s / (sm_ghz(r) * 8192e9)) if sm_ghz(r) else None}


def sm_ghz(r: dict):
    """Delivered compute capacity of the job: sum over ranks of applied SMs x
    median SM clock in the timed region (GHz).  Under the B200 power cap a
    full-SM rank clocks ~1.45-1.55 GHz while an SM-capped one holds ~1.95 GHz,
    so SM shares alone overstate a full B200 against a capped one; tokens/s per
    SM-GHz compares plans on what the hardware actually delivered."""
    ck = r.get("clocks") or {}
    clk = ck.get("sm_mhz_per_gpu") or {}
    ids = ck.get("gpu_of_rank") or []
    tot = 0.0
    for rank, (_, _, _, share) in enumerate(r.get("lin_per_rank") or []):
        mhz = clk.get(ids[rank]) if rank < len(ids) else None
        if mhz is None:
            return None
        tot += share * 148 * mhz / 1e3
    return tot or None


def reference_cost(name: str, seconds: float | None, speeds=None):
    """Predicted step time / MFU of the plan by the reference cost model
    (cost_model.cpp:210-265, restated in the executor: Plan.cost, parity with
    the compiled reference in tests/test_costmodel.py).  Mixed-speed TP plans,
    which the reference formula refuses, are priced by the labelled per-rank
    extension.  With `speeds` (closed-loop calibration) the
    cluster's peak_tflops are replaced by the measured per-device speeds and
    the calibrated prediction is compared with the measured step time."""
    from paper_2409_01143_b200 import calibrate
    from paper_2409_01143_b200.hexexec import HexexecError, Plan
    c, m, p, _ = load(name)
    out = {}
    try:
        r = Plan(c, m, p).cost(1.0)
        out = {"predicted_s": r["total"], "predicted_mfu": r["mfu"], "formula": "reference"}
    except HexexecError as e:
        r = Plan(c, m, p).cost(1.0, extension=True)
        out = {"predicted_s": r["total"], "predicted_mfu": r["mfu"],
               "formula": "extension (per-rank TP widths / speeds)", "reference_refuses": e.msg}
    if seconds:
        out["measured_s"] = seconds
    if speeds:
        cal = calibrate.calibrated_cluster(c, {d: v for d, v, _ in speeds},
                                           {d: f for d, _, f in speeds})
        rc = Plan(cal, m, p).cost(1.0, extension=True)
        out["calibrated"] = {
            "device_tflops": {d: round(v / 1e12, 1) for d, v, _ in speeds},
            "predicted_s": rc["total"], "breakdown_s": {k: rc[k] for k in (
                "compute", "tp_comm", "pp_comm", "dp_comm", "bubble")}}
        if seconds:
            out["calibrated"]["rel_error"] = (rc["total"] - seconds) / seconds
    return out


def cpu_reference(name: str, steps: int, warmup: int) -> dict:
    """See _cpu_reference.  BLAS threads are set to every host core explicitly:
    torchrun exports OMP_NUM_THREADS=1 to each rank, which would otherwise pin
    the numpy BLAS of the N > 1 reference arm to one core."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    import numpy  # noqa: F401  (threadpoolctl only sees BLAS libraries already loaded)
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        return _cpu_reference(name, steps, warmup)
    with threadpool_limits(limits=cores or 1, user_api="blas"):
        return _cpu_reference(name, steps, warmup)


def _cpu_reference(name: str, steps: int, warmup: int) -> dict:
    """The CPU reference of this path: the fp32 numpy oracle port
    (oracle/numeric.py; the reference repo has no numeric training step,
    SURVEY §0) on a bounded sample of the plan's workload, run as is: one
    sample (seq_len tokens) of the plan's model -- embedding, every decoder
    layer, final norm, LM head, CE, full backward -- per step, nothing
    extrapolated.  The AdamW update (once per global batch) is not part of the
    sample.  BLAS and the per-head attention loops use every host core.
    Loads only oracle/ code (numpy + the compiled reference planner)."""
    import numpy as np
    from oracle import bookkeeping as bk
    from oracle import numeric as O
    c, m, p, idx = load(name)
    md = bk.model_defaults(json.loads(m))
    cl = {"machines": {"box": {"intra_bandwidth_gbps": 900, "intra_latency_us": 3}},
          "devices": [{"id": "cpu", "machine": "box", "memory_gib": 64, "peak_tflops": 1}],
          "inter": {"bandwidth_gbps": 900, "latency_us": 3}}
    L_model = md["num_layers"]
    # deep models (the 32-layer 8-GPU workload): the bounded sample runs the
    # first MAX_REF_LAYERS layers (identical shapes) and the tokens/s of the
    # full model is extrapolated by training FLOPs -- labelled in the line
    L = min(L_model, MAX_REF_LAYERS)
    md_run = dict(md, num_layers=L)
    plan = {"global_batch": 1, "pipelines": [{"batch": 1, "micro_batch": 1, "stages": [
        {"devices": ["cpu"], "tp": 1, "layer_start": 0, "layer_count": L}]}]}
    t0 = time.perf_counter()
    st = O.Step(cl, md_run, json.dumps(plan))
    init_s = time.perf_counter() - t0
    stages = st.stage_parts(0)
    S = md["seq_len"]
    times = []
    G = {k: np.zeros_like(v) for k, v in st.W.items()}
    for i in range(warmup + steps):
        tok = st.tokens(i, 0, 1)
        t0 = time.perf_counter()
        st.micro_batch(tok, stages, S, G)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cores = cores or 1
    # the reference's own CPU path for the plan (SURVEY 8(d) "CPU reference
    # timing" (a)): hexplan_schedule on this config's cluster, compiled from the
    # reference sources (oracle/_ref), HEXPLAN_THREADS = host cores
    planner = None
    cost = None
    try:
        from oracle import refshim
        if refshim.available():
            kind = "symmetric" if idx["source"].endswith("symmetric") else "schedule"
            cfg = idx.get("config")
            if not cfg:  # hand plan: time the scheduler on its cluster
                cfg = {"global_batch": json.loads(p)["global_batch"], "iterations": 20,
                       "seed": 0, "threads": cores}
            t0 = time.perf_counter()
            res = refshim.plan(c, m, json.dumps(cfg), kind)
            planner = {"hexplan": kind, "wall_s": round(time.perf_counter() - t0, 4),
                       "found": bool(res.get("found")), "predicted_s": res.get("cost"),
                       "config": cfg}
            # the reference cost model (iteration_time, cost_model.cpp:210-258) on
            # the executed plan itself, through the compiled reference
            chk = refshim.check_plan(c, m, p)
            cost = ({"predicted_s": chk["cost"]["total"], "predicted_mfu": chk["cost"]["mfu"],
                     "source": "oracle/_ref iteration_time"} if "cost" in chk else
                    {"reference_refuses": chk.get("cost_error"),
                     "source": "oracle/_ref iteration_time"})
    except Exception as e:  # noqa: BLE001  (reported, never fatal for the bench)
        planner = {"error": str(e)[:200]}
    t = statistics.mean(times)
    factor = 1.0
    if L < L_model:
        _, f_run = model_flops(md_run, S)
        _, f_all = model_flops(md, S)
        factor = f_run / f_all
    what = (f"the whole {L}-layer model" if L == L_model else
            f"embedding + the first {L} of {L_model} layers + final norm, LM head")
    out = {"value": S / t * factor, "unit": "tokens/s", "cores": cores, "kind": "port",
           "reference_planner": planner, "reference_cost_model": cost,
           "sample": (f"numpy fp32 oracle (oracle/numeric.py): per step one sample of "
                      f"{S} tokens through {what} (CE; forward + backward), measured; "
                      f"AdamW excluded; mean of {steps} after {warmup} warm-up; BLAS + "
                      f"per-head threads = {cores} host cores"),
           "sample_ms": [round(x * 1e3, 1) for x in times], "init_s": round(init_s, 1),
           "ms_per_sample": t * 1e3}
    if L < L_model:
        out["extrapolation"] = {"layers_run": L, "layers": L_model,
                                "measured_unit_tokens_per_s": S / t,
                                "training_flop_ratio": factor,
                                "note": "value = measured unit rate x (unit FLOPs / full-model FLOPs)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--plan", default=None, help="configs/plans/<name>.json (asymmetric arm)")
    ap.add_argument("--even-plans", default=None,
                    help="comma-separated even-split comparison plans ('none' to skip)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the extra asymmetric arms")
    ap.add_argument("--exec-config", default="{}", help="JSON executor config overrides")
    a = ap.parse_args()
    EXEC_CFG.update(json.loads(a.exec_config))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != a.gpus and "RANK" in os.environ:
        raise SystemExit(f"WORLD_SIZE {world} != --gpus {a.gpus}")
    asym, even = PLANS.get(a.gpus, (None, None))
    if a.plan:
        asym = a.plan
        even = None
    if a.even_plans:
        even = None if a.even_plans == "none" else a.even_plans
    if asym is None:
        raise SystemExit(f"no default plan for {a.gpus} GPUs; pass --plan")
    _, m_doc, _, _ = load(asym)
    model = json.loads(m_doc)
    config = {"workload": f"{asym}: {INDEX_DESC.get(asym, asym)}", "plan": asym,
              "model": model, "global_batch": json.loads(load(asym)[2])["global_batch"],
              "seq_len": model["seq_len"], "even_split_plan": even,
              "l2": "working set per step >> 126 MB L2 (weights + optimizer state + activations)",
              "parallelism": "plan-defined asymmetric DP/PP/TP, one process per GPU"}
    if EXEC_CFG:
        config["exec_config"] = dict(EXEC_CFG)

    if a.impl == "reference":
        # the reference arm: the CPU oracle port on the host cores, rank 0 only;
        # nothing from the product package is imported or loaded here
        if rank != 0:
            return
        ref = cpu_reference(asym, steps=a.steps, warmup=a.warmup)
        line = {"metric": METRIC, "value": ref["value"], "unit": "tokens/s", "impl": "reference",
                "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
                "ms_per_step": ref["ms_per_sample"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": config,
                "step_unit": "one sample (seq_len tokens) of the plan's model, fwd + bwd",
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                     "reference_planner", "sample_ms", "init_s",
                                                     "extrapolation") if k in ref},
                "e2e": {"value": ref["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "reference_cost_model": ref["reference_cost_model"]}
        print(json.dumps(line), flush=True)
        return

    pk = peaks()
    r = run_plan(asym, a.steps, a.warmup, rank, world, clocks=(rank == 0))
    s = summarize(r, a.steps, pk)
    ev = None
    alts = []
    for a_name in (ALT.get(a.gpus, "").split(",") if not a.plan and not a.no_alt else []):
        if a_name:
            ra = run_plan(a_name, a.steps, a.warmup, rank, world, clocks=(rank == 0))
            alts.append(dict(summarize(ra, a.steps, pk), clocks=ra["clocks"]))
    evs = []
    for e_name in (even.split(",") if even else []):
        re_ = run_plan(e_name, a.steps, a.warmup, rank, world, clocks=(rank == 0))
        evs.append(dict(summarize(re_, a.steps, pk), clocks=re_["clocks"]))
    ev = evs[0] if evs else None
    if rank != 0:
        return
    # roofline of the TP GEMMs on rank 0 (the full-SM rank of every default plan);
    # each rank's peak is its applied SM share x the sustained tensor peak
    f0, ms0, n0, sh0 = r["lin_per_rank"][0]
    lin_ms_launch = ms0 / max(n0, 1)
    lin_flops_launch = f0 / max(n0, 1)
    achieved = lin_flops_launch / (lin_ms_launch / 1e3) / 1e12 if lin_ms_launch > 0 else None
    peak0 = pk["bf16_tflops_sustained"] * sh0
    per_rank_roof = [{"rank": i, "sm_share": round(sh, 4),
                      "achieved_tflops": (fl / (ms / 1e3) / 1e12) if ms > 0 else None,
                      "frac_of_share_peak": (fl / (ms / 1e3) / 1e12 / (pk["bf16_tflops_sustained"] * sh))
                      if ms > 0 and sh > 0 else None}
                     for i, (fl, ms, nl_, sh) in enumerate(r["lin_per_rank"])]
    # DRAM bytes per TP-GEMM launch (read + write) from one ncu --set full
    # capture of the step's twelve linear GEMM shapes (scripts/gemm_traffic_probe.py,
    # launch-weighted like `achieved`), beside their algorithmic bytes
    traffic, traffic_alg = None, None
    for tf in (os.path.join(ROOT, "profiles", "r02_gemm_traffic.json"),
               os.path.join(ROOT, "profiles", "gemm_traffic.json")):
        if os.path.exists(tf):
            tj = json.load(open(tf))
            traffic, traffic_alg = tj.get("bytes_per_launch"), tj.get("algorithmic_bytes_per_launch")
            break
    cpu = None
    if a.gpus == 1 and not a.no_cpu_baseline:
        cb = cpu_reference(asym, steps=1, warmup=0)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "reference_planner",
                                  "reference_cost_model", "extrapolation") if k in cb}
    line = {
        "metric": METRIC, "value": s["tokens_per_s"], "unit": "tokens/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": s["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens (counter RNG), random-init weights (N(0,0.02) Irwin-Hall)",
        "config": config,
        "mfu": {"ref_convention": s["mfu_ref_convention"], "exact": s["mfu_exact"],
                "peak_per_rank": f"sm_share x {pk['bf16_tflops']} TFLOPS ({pk['source']})",
                "aggregate_sm_share": s["aggregate_sm_share"]},
        "even_split": ev,
        "even_split_other": evs[1:],
        "asym_other": alts,
        "sm_ghz": s["sm_ghz"], "tokens_per_s_per_sm_ghz": s["tokens_per_s_per_sm_ghz"],
        "mfu_gap_vs_even": (ev["mfu_ref_convention"] - s["mfu_ref_convention"]) if ev else None,
        "mfu_gap_vs_even_rel": (1 - s["mfu_ref_convention"] / ev["mfu_ref_convention"]) if ev else None,
        "mfu_at_delivered_clock": s["mfu_at_delivered_clock"],
        "mfu_gap_vs_even_at_delivered_clock_rel": (
            1 - s["mfu_at_delivered_clock"] / ev["mfu_at_delivered_clock"])
        if ev and ev.get("mfu_at_delivered_clock") and s["mfu_at_delivered_clock"] else None,
        "e2e": {"value": s["e2e_tokens_per_s"], "unit": "tokens/s",
                "h2d_bytes_per_step": int(r["h2d"]), "d2h_bytes_per_step": int(r["d2h"])},
        "gpu_launches": int(r["launches"] * a.steps),
        "roofline": {"bound": "tensor", "kernel": "tcgen05 TP GEMMs (QKV/O/gate-up/down, fwd+dgrad+wgrad)",
                     "achieved": achieved, "peak": peak0, "unit": "TFLOP/s",
                     "frac": achieved / peak0 if achieved else None,
                     "peak_kind": "sustained (kernel timed inside a long step) x rank 0 SM share",
                     "rank": 0, "per_rank": per_rank_roof,
                     "timing": ("CUDA events captured around every GEMM in the step graph, "
                                "last timed replay" if r.get("gemm_graph") else
                                "CUDA events around every GEMM, eager profiled pass"),
                     # the graph events bracket one micro-batch's GEMMs; a step
                     # runs n_mb micro-batches of the same launches
                     "launches_sampled": n0,
                     "micro_batches_sampled": 1 if r.get("gemm_graph") else None,
                     "launches_per_step": (n0 * r["n_mb"][0]) if r.get("gemm_graph") else n0 / max(
                         r["stats"].get("gemm_profile", {}).get("steps", 1), 1),
                     "algorithmic_flops_per_launch": lin_flops_launch,
                     "avg_launch_ms": lin_ms_launch, "traffic": traffic,
                     "traffic_algorithmic_bytes": traffic_alg},
        "gemm_profile_rank0": r.get("gemm_graph") or r["stats"].get("gemm_profile"),
        "phase_ms_rank0": r["stats"].get("ms"),
        "timeline_ms_rank0_profiled": r["stats"].get("timeline_ms"),
        "timeline_ms_per_step_per_rank_profiled": r["tl_all"] if a.gpus > 1 else None,
        "timeline_ms_one_microbatch_per_rank_graph": r["tlg_all"],
        "sm_cap_per_rank": r["sm_caps"],
        "clocks": r["clocks"],
        # e2e steps sync the host every step: the GPU idles for the copy / sync
        # gap, and under the power cap the SM clock recovers a little, which is
        # why e2e can come out at or above the back-to-back device-timed value
        "clocks_e2e": r["clocks_e2e"],
        "value_second_device_pass_after_e2e": (
            json.loads(load(asym)[2])["global_batch"] * model["seq_len"] * a.steps / (r["dev2_ms"] / 1e3)),
        "cpu_baseline": cpu,
        "reference_cost_model": reference_cost(asym, s["ms_per_step"] / 1e3, r.get("speeds")),
        "loss": s["loss"],
    }
    print(json.dumps(line), flush=True)


INDEX_DESC = {
    "llama7b_4l_1gpu": "Llama-7B-shaped 4-layer block, seq 2048, global batch 8, one B200 (tp=1)",
    "llama7b_4l_tp31": "Llama-7B-shaped 4-layer block, seq 2048, TP=2 widths 3:1 on 2xB200, "
                       "rank 1 SM-capped to 1/3",
    "llama7b_4l_4_asym": "Llama-7B-shaped 4-layer block, hexplan_schedule plan on 4xB200 "
                         "tiers [F,F,1/2,1/2]",
    "llama7b_8_asym": "Llama-7B (32 layers) on 8xB200 tiers [F,F,F,F,1/2,1/2,1/3,1/3]: "
                      "hexplan_schedule plan, asymmetric DP 15/12/12/12/13",
    "llama7b_4l_4_cal": "Llama-7B-shaped 4-layer block, hexplan_schedule plan on 4xB200 tiers "
                        "[F,F,1/2,1/2] with calibrated tier speeds: asymmetric DP 14/14/10/10",
    "llama7b_8_cal": "Llama-7B (32 layers) on 8xB200 tiers [F,F,F,F,1/2,1/2,1/3,1/3] with "
                     "calibrated tier speeds: hexplan_schedule plan, asymmetric DP 21/21/22 over "
                     "PP 16/16, 16/16 and TP=2 stages 20/12",
    "llama13b_pp3_asymtp": "Llama-13B 3-stage pipeline 16/14/10, asymmetric TP inside stages",
    "llama30b_8_tiers": "Llama-30B layers under a full hexplan_schedule plan, 8xB200 SM-capped tiers",
}

if __name__ == "__main__":
    main()
