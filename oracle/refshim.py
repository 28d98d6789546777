"""ORACLE TEST INFRASTRUCTURE — ctypes access to the compiled reference.

oracle/_ref/libhexplan_ref.so is built by oracle/Makefile from the reference
sources under /root/reference/proj/src (plus oracle/ref_shim.cpp).  It exposes
the reference's own C ABI (proj/include/hexplan.h) and the shim's
hexref_check_plan / hexref_mfu.  Tests that need it skip when it is absent
(e.g. on a GPU box where it was not shipped).
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libhexplan_ref.so")


def available() -> bool:
    return os.path.exists(LIB)


_lib = None


def lib():
    global _lib
    if _lib is None:
        l = C.CDLL(LIB)
        vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
        for name, res, args in [
            ("hexplan_cluster_parse", C.c_int, [cp, C.POINTER(vp), cp, sz]),
            ("hexplan_model_parse", C.c_int, [cp, C.POINTER(vp), cp, sz]),
            ("hexplan_cluster_free", None, [vp]),
            ("hexplan_model_free", None, [vp]),
            ("hexplan_schedule", C.c_int, [vp, vp, cp, C.POINTER(vp), cp, sz]),
            ("hexplan_symmetric_baseline", C.c_int, [vp, vp, cp, C.POINTER(vp), cp, sz]),
            ("hexplan_oracle", C.c_int, [vp, vp, cp, C.POINTER(vp), cp, sz]),
            ("hexplan_result_found", C.c_int, [vp]),
            ("hexplan_result_cost", C.c_double, [vp]),
            ("hexplan_result_mfu", C.c_double, [vp]),
            ("hexplan_result_plan_json", vp, [vp]),
            ("hexplan_result_report_json", vp, [vp]),
            ("hexplan_result_free", None, [vp]),
            ("hexplan_string_free", None, [vp]),
            ("hexref_check_plan", C.c_int, [cp, cp, cp, C.POINTER(vp), cp, sz]),
            ("hexref_mfu", C.c_double, [cp, cp, C.c_double, C.c_longlong]),
            ("hexref_free", None, [vp]),
        ]:
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _take(ptr, free):
    if not ptr:
        return None
    s = C.cast(ptr, C.c_char_p).value.decode()
    free(ptr)
    return s


def check_plan(cluster: str, model: str, plan: str) -> dict:
    """num_micro_batches, rebuilt dp_groups, validate message, cost report /
    cost_error, serialize_plan bytes — all computed by reference code."""
    l = lib()
    out = C.c_void_p()
    err = C.create_string_buffer(512)
    st = l.hexref_check_plan(cluster.encode(), model.encode(), plan.encode(), C.byref(out),
                             err, len(err))
    if st != 0:
        raise ValueError(err.value.decode())
    return json.loads(_take(out, l.hexref_free))


def mfu(cluster: str, model: str, seconds: float, global_batch: int) -> float:
    return lib().hexref_mfu(cluster.encode(), model.encode(), seconds, global_batch)


def plan(cluster: str, model: str, config: str, kind: str = "schedule") -> dict:
    """Run hexplan_schedule / hexplan_symmetric_baseline / hexplan_oracle."""
    l = lib()
    c, m, r = C.c_void_p(), C.c_void_p(), C.c_void_p()
    err = C.create_string_buffer(512)
    assert l.hexplan_cluster_parse(cluster.encode(), C.byref(c), err, len(err)) == 0, err.value
    assert l.hexplan_model_parse(model.encode(), C.byref(m), err, len(err)) == 0, err.value
    fn = {"schedule": l.hexplan_schedule, "symmetric": l.hexplan_symmetric_baseline,
          "oracle": l.hexplan_oracle}[kind]
    st = fn(c, m, config.encode(), C.byref(r), err, len(err))
    try:
        if st != 0:
            raise ValueError(f"status {st}: {err.value.decode()}")
        res = {"found": l.hexplan_result_found(r), "cost": l.hexplan_result_cost(r),
               "mfu": l.hexplan_result_mfu(r),
               "plan": _take(l.hexplan_result_plan_json(r), l.hexplan_string_free),
               "report": _take(l.hexplan_result_report_json(r), l.hexplan_string_free)}
        return res
    finally:
        if r:
            l.hexplan_result_free(r)
        l.hexplan_model_free(m)
        l.hexplan_cluster_free(c)
