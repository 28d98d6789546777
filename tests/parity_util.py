"""Shared helpers of the GPU parity tests: launch a plan's ranks (one process
per GPU, tests/rank_worker.py), or run a one-GPU plan in-process; compute the
CPU fp32 oracle (oracle/numeric.py, test infrastructure) on the same seeds and
tokens; compare normwise.

Tolerance (BASELINE north star): bf16 tensor-core accumulation vs the fp32
oracle, rtol 2e-2, normwise per tensor (||x - ref|| / ||ref||) for reduced
gradients and updated weights, relative for the loss."""
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = os.path.join(ROOT, "configs")
INDEX = json.load(open(os.path.join(CFG, "index.json")))
RTOL = 2e-2


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_plan(name, tmp_path, steps=1, xcfg=None, host_tokens=True, timeout=600, read=None,
             env=None):
    for attempt in range(3):  # a rendezvous port taken between probe and bind: retry
        try:
            return _run_plan(name, tmp_path, steps, xcfg, host_tokens, timeout, read, env)
        except PortInUse:
            continue
    raise RuntimeError("no free rendezvous port")


class PortInUse(Exception):
    pass


def world_of(name):
    e = INDEX[name]
    return len(json.load(open(os.path.join(CFG, "clusters", e["cluster"] + ".json")))["devices"])


def _run_plan(name, tmp_path, steps, xcfg, host_tokens, timeout, read=None, env_extra=None):
    world = world_of(name)
    if ngpu() < world:
        pytest.skip(f"{name} needs {world} GPUs")
    os.makedirs(tmp_path, exist_ok=True)
    port = free_port()
    procs, logs = [], []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        if read:
            env["HEXEXEC_TEST_READ"] = read
        env.update(env_extra or {})
        logs.append(open(os.path.join(tmp_path, f"rank{r}.err"), "w+"))
        procs.append(subprocess.Popen(
            [sys.executable, os.path.join(ROOT, "tests", "rank_worker.py"), name, str(tmp_path),
             str(steps), json.dumps(xcfg or {}), "1" if host_tokens else "0"], env=env,
            stderr=logs[-1]))
    t0 = time.time()
    while any(p.poll() is None for p in procs):
        if any(p.poll() not in (None, 0) for p in procs) or time.time() - t0 > timeout:
            time.sleep(2)  # let the others report, then stop them
            for p in procs:
                if p.poll() is None:
                    p.kill()
            break
        time.sleep(0.2)
    for p in procs:
        p.wait()
    errs = []
    for lg in logs:
        lg.seek(0)
        errs.append(lg.read())
        lg.close()
    if any(p.returncode != 0 for p in procs):
        if any("EADDRINUSE" in e for e in errs):
            raise PortInUse()
        sys.stderr.write("\n".join(errs))
    assert all(p.returncode == 0 for p in procs), [p.returncode for p in procs]
    out = []
    for r in range(world):
        f = os.path.join(tmp_path, f"rank{r}.npz")
        with np.load(f) as z:
            out.append({k: z[k] for k in z.files})
        os.remove(f)  # the large-shape plans write several GB per rank
    return out


_ORACLE = {}


def oracle_step(name, **kw):
    from oracle import numeric as O
    e = INDEX[name]
    c = json.load(open(os.path.join(CFG, "clusters", e["cluster"] + ".json")))
    m = json.load(open(os.path.join(CFG, "models", e["model"] + ".json")))
    return O.Step(c, m, open(os.path.join(CFG, "plans", name + ".json")).read(), **kw)


def oracle_for(name, keep=True, bf16_points=False):
    """(loss, reduced grads, updated weights) of step 0 by the fp32 oracle
    (bf16_points: with the executor's bf16 storage points emulated).
    keep=False: not cached (the large-shape plans hold 3-5 GB per copy)."""
    key = (name, bf16_points)
    if key in _ORACLE:
        return _ORACLE[key]
    st = oracle_step(name, bf16_points=bf16_points)
    loss, G, W = st.run(0)
    st.mom = st.vel = None
    out = (loss, G, W)
    if keep:
        _ORACLE[key] = out
    return out


def torch_floor(name, G, dtype="bf16"):
    """Per-tensor normwise deviation from the oracle gradients G of the same
    step in plain PyTorch (tests/torch_bf16_ref.py) on cuda:0: dtype "bf16"
    = torch.autocast-style bf16 (the bf16 floor), "fp32" = an independent
    fp32 restatement that pins the oracle.  Returns (loss, {tensor: error})."""
    import torch_bf16_ref as TR
    loss, Gt = TR.step_grads(oracle_step(name), dtype=dtype)
    out = {t: rel(Gt[t], G[t]) for t in G}
    del Gt
    import torch
    torch.cuda.empty_cache()
    return loss, out


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def check_against_oracle(name, ranks, oracle=None, report=None):
    """Every rank's loss, and every reduced gradient / updated weight it holds,
    against the oracle's rows of that tensor; every tensor held somewhere.
    report: dict filled with the worst relative error per tensor.  All
    tensors are compared before anything is asserted (the failure message
    lists every tensor out of tolerance)."""
    loss, G, W = oracle or oracle_for(name)
    seen = set()
    rep = {} if report is None else report
    for r in ranks:
        for key in r:
            if not key.endswith("|grad"):
                continue
            t = key[:-5]
            row0 = int(r[t + "|row0"])
            g = r[key]
            eg = rel(g, G[t][row0:row0 + g.shape[0]])
            ew = rel(r[t + "|w"], W[t][row0:row0 + g.shape[0]])
            o = rep.setdefault(t, [0.0, 0.0])
            o[0], o[1] = max(o[0], eg), max(o[1], ew)
            seen.add(t)
    bad = {t: v for t, v in rep.items() if v[0] >= RTOL or v[1] >= RTOL}
    if bad:
        print("PARITY-REPORT " + json.dumps({t: [round(a, 5), round(b, 5)]
                                              for t, (a, b) in sorted(rep.items())}))
    for r in ranks:
        assert abs(float(r["losses"][0]) - loss) <= RTOL * abs(loss), (r["losses"][0], loss)
    assert not bad, bad
    assert seen == set(G), set(G) - seen  # every tensor is held somewhere


def run_inprocess(name, steps=1, xcfg=None, read=None):
    """A one-GPU plan through the public API in this process (no npz round
    trip): returns the same dict as one rank of run_plan."""
    import re
    from paper_2409_01143_b200 import Executor
    if ngpu() < 1:
        pytest.skip("no CUDA device")
    e = INDEX[name]
    c = open(os.path.join(CFG, "clusters", e["cluster"] + ".json")).read()
    m = open(os.path.join(CFG, "models", e["model"] + ".json")).read()
    p = open(os.path.join(CFG, "plans", name + ".json")).read()
    ex = Executor(c, m, p, xcfg or {}, rank=0, world_size=1, device=0)
    try:
        res, losses = {}, []
        for s in range(steps):
            losses.append(ex.step(ex.synth_tokens(s)))
            if s == 0:
                for t in ex.role["tensors"]:
                    if read and not re.search(read, t["name"]):
                        continue
                    res[t["name"] + "|grad"] = ex.read(t["name"], 1)
                    res[t["name"] + "|w"] = ex.read(t["name"], 0)
                    res[t["name"] + "|row0"] = np.int64(t["row0"])
        res["losses"] = np.array(losses, np.float64)
        res["stats"] = np.frombuffer(json.dumps(ex.stats()).encode(), np.uint8)
        return res
    finally:
        ex.close()
