"""Python mirror of include/hexexec.h.

Same call shapes as the reference's C ABI conventions
(/root/reference/proj/include/hexplan.h: opaque handle + status + err buffer),
raised as HexexecError carrying the status code.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Optional

import numpy as np

from . import _lib as L
from ._lib import HexexecError  # noqa: F401


def _b(s: Optional[str]):
    return None if s is None else s.encode()


class Plan:
    """Parsed + validated plan with its rank layout (host only)."""

    def __init__(self, cluster_json: str, model_json: str, plan_json: str):
        h = C.c_void_p()
        err = L.errbuf()
        L.check(L.hexexec_plan_parse(_b(cluster_json), _b(model_json), _b(plan_json),
                                     C.byref(h), err, len(err)), err)
        self._h = h

    def serialize(self) -> str:
        return L.take_string(L.hexexec_plan_serialize(self._h))

    def layout(self) -> dict:
        return json.loads(L.take_string(L.hexexec_plan_layout_json(self._h)))

    @property
    def world_size(self) -> int:
        return L.hexexec_plan_world_size(self._h)

    def cost(self, state_multiplier: float = 1.0, extension: bool = False) -> dict:
        """Reference cost model (cost_model.cpp:210-258) on this plan; with
        extension=True uneven / mixed-speed TP stages are priced per rank."""
        out = C.c_void_p()
        err = L.errbuf()
        L.check(L.hexexec_plan_cost(self._h, state_multiplier, 1 if extension else 0,
                                    C.byref(out), err, len(err)), err)
        return json.loads(L.take_string(out))

    def mfu(self, seconds: float) -> float:
        """Reference-convention MFU (cost_model.cpp:260-265) of a step time."""
        return L.hexexec_plan_mfu(self._h, seconds)

    def close(self):
        if self._h:
            L.hexexec_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unique_id() -> bytes:
    n = L.hexexec_unique_id_size()
    buf = C.create_string_buffer(n)
    err = L.errbuf()
    L.check(L.hexexec_unique_id(buf, n, err, len(err)), err)
    return buf.raw


class Executor:
    """One executor rank (one process per GPU)."""

    def __init__(self, cluster_json: str, model_json: str, plan_json: str,
                 exec_config: dict | str | None = None, rank: int = 0, world_size: int = 1,
                 device: int = 0, uid: bytes | None = None):
        if isinstance(exec_config, dict):
            exec_config = json.dumps(exec_config)
        h = C.c_void_p()
        err = L.errbuf()
        uid_buf = C.create_string_buffer(uid, len(uid)) if uid else None
        L.check(L.hexexec_ctx_create(_b(cluster_json), _b(model_json), _b(plan_json),
                                     _b(exec_config or ""), rank, world_size, device,
                                     uid_buf, len(uid) if uid else 0, C.byref(h), err,
                                     len(err)), err)
        self._h = h
        self.layout = Plan(cluster_json, model_json, plan_json).layout()
        self.rank = rank
        self.role = self.layout["ranks"][rank]

    def step(self, tokens: Optional[np.ndarray] = None) -> float:
        """One training step; tokens = this pipeline's [batch, S+1] int32 (host)."""
        loss = C.c_float(0.0)
        err = L.errbuf()
        if tokens is None:
            L.check(L.hexexec_step(self._h, None, 0, C.byref(loss), err, len(err)), err)
        else:
            t = np.ascontiguousarray(tokens, dtype=np.int32)
            L.check(L.hexexec_step(self._h, t.ctypes.data, t.size, C.byref(loss), err,
                                   len(err)), err)
        return float(loss.value)

    def step_async(self):
        err = L.errbuf()
        L.check(L.hexexec_step_async(self._h, err, len(err)), err)

    def sync(self):
        err = L.errbuf()
        L.check(L.hexexec_sync(self._h, err, len(err)), err)

    def set_profile(self, on: bool):
        L.check(L.hexexec_set_profile(self._h, 1 if on else 0), None, "set_profile")

    def timer_start(self):
        err = L.errbuf()
        L.check(L.hexexec_timer(self._h, 0, None, err, len(err)), err)

    def timer_stop(self) -> float:
        ms = C.c_float(0.0)
        err = L.errbuf()
        L.check(L.hexexec_timer(self._h, 1, C.byref(ms), err, len(err)), err)
        return float(ms.value)

    def last_loss(self) -> float:
        loss = C.c_float(0.0)
        err = L.errbuf()
        L.check(L.hexexec_last_loss(self._h, C.byref(loss), err, len(err)), err)
        return float(loss.value)

    def synth_tokens(self, step: int) -> np.ndarray:
        r = self.role
        if not r["active"]:
            return np.zeros((0, 0), np.int32)
        b = r["samples"][1] - r["samples"][0]
        S = self.layout["model"]["seq_len"]
        out = np.zeros((b, S + 1), np.int32)
        err = L.errbuf()
        L.check(L.hexexec_synth_tokens(self._h, step, out.ctypes.data, out.size, err,
                                       len(err)), err)
        return out

    def tensor_info(self, name: str):
        r0, rows, cols, grows = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        st = L.hexexec_tensor_info(self._h, _b(name), C.byref(r0), C.byref(rows),
                                   C.byref(cols), C.byref(grows))
        L.check(st, None, f"unknown tensor {name}")
        return r0.value, rows.value, cols.value, grows.value

    def read(self, name: str, which: int = 0) -> np.ndarray:
        """which: 0 master weights, 1 reduced gradient, 2 adam m, 3 adam v."""
        r0, rows, cols, _ = self.tensor_info(name)
        out = np.zeros((rows, cols), np.float32)
        if rows == 0:
            return out
        err = L.errbuf()
        L.check(L.hexexec_read_tensor(self._h, _b(name), which, out.ctypes.data, out.size,
                                      err, len(err)), err)
        return out

    def sm_probe(self, what: int, n: int) -> np.ndarray:
        """SM ids used by this rank's work: 0 = probe CTAs on the executor
        stream, 1 = on the comm stream, 2 = one persistent GEMM's CTAs."""
        out = np.full(n, -1, np.int32)
        written = C.c_int(0)
        err = L.errbuf()
        L.check(L.hexexec_sm_probe(self._h, what, out.ctypes.data, n, C.byref(written), err,
                                   len(err)), err)
        return out[:written.value]

    def stats(self) -> dict:
        return json.loads(L.take_string(L.hexexec_stats_json(self._h)) or "{}")

    def close(self):
        if getattr(self, "_h", None):
            L.hexexec_ctx_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
