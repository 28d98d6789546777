"""ctypes binding of include/hexexec.h (the product's C ABI).

The shared library is built in-tree (paper_2409_01143_b200/libhexexec.so).
There is no fallback: if it is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhexexec.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

OK, ERR_PARSE, ERR_INVALID, ERR_INFEASIBLE, ERR_LIMIT, ERR_INTERNAL, ERR_CUDA, ERR_NCCL = range(8)
STATUS_NAMES = {0: "OK", 1: "PARSE", 2: "INVALID", 3: "INFEASIBLE", 4: "LIMIT",
                5: "INTERNAL", 6: "CUDA", 7: "NCCL"}

_c = C.c_char_p
_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_f = C.c_float
_sz = C.c_size_t
_st = C.c_int


def _sig(name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


# plan / bookkeeping
hexexec_plan_parse = _sig("hexexec_plan_parse", _st, _c, _c, _c, C.POINTER(_vp), _c, _sz)
hexexec_plan_serialize = _sig("hexexec_plan_serialize", _vp, _vp)
hexexec_plan_layout_json = _sig("hexexec_plan_layout_json", _vp, _vp)
hexexec_plan_world_size = _sig("hexexec_plan_world_size", _i, _vp)
hexexec_plan_cost = _sig("hexexec_plan_cost", _st, _vp, C.c_double, _i, C.POINTER(_vp), _c, _sz)
hexexec_plan_mfu = _sig("hexexec_plan_mfu", C.c_double, _vp, C.c_double)
hexexec_plan_free = _sig("hexexec_plan_free", None, _vp)
# nccl
hexexec_unique_id_size = _sig("hexexec_unique_id_size", _sz)
hexexec_unique_id = _sig("hexexec_unique_id", _st, _vp, _sz, _c, _sz)
# executor
hexexec_ctx_create = _sig("hexexec_ctx_create", _st, _c, _c, _c, _c, _i, _i, _i, _vp, _sz,
                          C.POINTER(_vp), _c, _sz)
hexexec_ctx_free = _sig("hexexec_ctx_free", None, _vp)
hexexec_step = _sig("hexexec_step", _st, _vp, _vp, _sz, C.POINTER(_f), _c, _sz)
hexexec_step_async = _sig("hexexec_step_async", _st, _vp, _c, _sz)
hexexec_sync = _sig("hexexec_sync", _st, _vp, _c, _sz)
hexexec_last_loss = _sig("hexexec_last_loss", _st, _vp, C.POINTER(_f), _c, _sz)
hexexec_timer = _sig("hexexec_timer", _st, _vp, _i, C.POINTER(_f), _c, _sz)
hexexec_set_profile = _sig("hexexec_set_profile", _st, _vp, _i)
hexexec_synth_tokens = _sig("hexexec_synth_tokens", _st, _vp, _i64, _vp, _sz, _c, _sz)
hexexec_tensor_info = _sig("hexexec_tensor_info", _st, _vp, _c, C.POINTER(_i64),
                           C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64))
hexexec_read_tensor = _sig("hexexec_read_tensor", _st, _vp, _c, _i, _vp, _sz, _c, _sz)
hexexec_stats_json = _sig("hexexec_stats_json", _vp, _vp)
hexexec_sm_probe = _sig("hexexec_sm_probe", _st, _vp, _i, _vp, _i, C.POINTER(_i), _c, _sz)
# kernels
hexexec_k_gemm = _sig("hexexec_k_gemm", _st, _i, _i, _i, _i, _i, _vp, _i, _i64, _i64, _i64,
                      _vp, _i, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i, _i, _f, _i, _vp)
hexexec_k_gemm_split = _sig("hexexec_k_gemm_split", _st, _i, _vp, _sz, _vp, _i)
hexexec_k_gemm_peers = _sig("hexexec_k_gemm_peers", _st, C.POINTER(_vp), _i)
hexexec_k_gemm_raster = _sig("hexexec_k_gemm_raster", _st, _i)
hexexec_k_gemm_sm_limit = _sig("hexexec_k_gemm_sm_limit", _st, _i)
hexexec_k_gemm_multicast = _sig("hexexec_k_gemm_multicast", _st, _i)
hexexec_k_gemm_tile_auto = _sig("hexexec_k_gemm_tile_auto", _st, _i)
hexexec_k_attn_variant = _sig("hexexec_k_attn_variant", _st, _i, _i)
hexexec_k_attn_fwd = _sig("hexexec_k_attn_fwd", _st, _vp, _vp, _vp, _i, _i, _i, _i, _f, _vp)
hexexec_k_attn_bwd = _sig("hexexec_k_attn_bwd", _st, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i,
                          _i, _i, _f, _vp)
hexexec_k_rmsnorm_fwd = _sig("hexexec_k_rmsnorm_fwd", _st, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i,
                             _f, _vp)
hexexec_k_rmsnorm_bwd = _sig("hexexec_k_rmsnorm_bwd", _st, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                             _vp, _vp, _i, _i, _vp)
hexexec_k_rope = _sig("hexexec_k_rope", _st, _vp, _i, _i, _i, _i, _f, _i, _vp)
hexexec_k_softmax_fwd = _sig("hexexec_k_softmax_fwd", _st, _vp, _vp, _i, _i, _vp)
hexexec_k_softmax_bwd = _sig("hexexec_k_softmax_bwd", _st, _vp, _vp, _vp, _f, _i, _i, _vp)
hexexec_k_swiglu_fwd = _sig("hexexec_k_swiglu_fwd", _st, _vp, _vp, _i, _i, _vp)
hexexec_k_swiglu_bwd = _sig("hexexec_k_swiglu_bwd", _st, _vp, _vp, _vp, _i, _i, _vp)
hexexec_k_ce = _sig("hexexec_k_ce", _st, _vp, _i, _i, _vp, _i, _i, _f, _vp, _vp, _vp, _vp)
hexexec_k_adamw = _sig("hexexec_k_adamw", _st, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _f, _f, _f,
                       _f, _f, _f, _i, _vp)
hexexec_k_init_normal = _sig("hexexec_k_init_normal", _st, _vp, _i64, _i64, _u64, _vp)
hexexec_k_tokens = _sig("hexexec_k_tokens", _st, _vp, _i64, _i, _i64, _u64, _i64, _i, _vp)
hexexec_k_sync = _sig("hexexec_k_sync", _st, _c, _sz)
hexexec_version = _sig("hexexec_version", _c)
hexexec_string_free = _sig("hexexec_string_free", None, _vp)

EXPORTED = [
    "hexexec_plan_parse", "hexexec_plan_serialize", "hexexec_plan_layout_json",
    "hexexec_plan_world_size", "hexexec_plan_cost", "hexexec_plan_mfu", "hexexec_plan_free", "hexexec_unique_id_size",
    "hexexec_unique_id", "hexexec_ctx_create", "hexexec_ctx_free", "hexexec_step",
    "hexexec_step_async", "hexexec_sync", "hexexec_last_loss", "hexexec_timer",
    "hexexec_set_profile",
    "hexexec_synth_tokens",
    "hexexec_tensor_info", "hexexec_read_tensor", "hexexec_stats_json", "hexexec_sm_probe", "hexexec_k_gemm", "hexexec_k_gemm_split",
    "hexexec_k_gemm_peers", "hexexec_k_gemm_raster", "hexexec_k_gemm_sm_limit",
    "hexexec_k_gemm_multicast", "hexexec_k_gemm_tile_auto",
    "hexexec_k_attn_variant", "hexexec_k_attn_fwd", "hexexec_k_attn_bwd",
    "hexexec_k_rmsnorm_fwd", "hexexec_k_rmsnorm_bwd", "hexexec_k_rope", "hexexec_k_softmax_fwd",
    "hexexec_k_softmax_bwd", "hexexec_k_swiglu_fwd", "hexexec_k_swiglu_bwd", "hexexec_k_ce",
    "hexexec_k_adamw", "hexexec_k_init_normal", "hexexec_k_tokens", "hexexec_k_sync",
    "hexexec_version", "hexexec_string_free",
]


class HexexecError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hexexec {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg


def take_string(ptr) -> str | None:
    """Copy a library-owned malloc'd string and free it."""
    if not ptr:
        return None
    s = C.cast(ptr, C.c_char_p).value.decode()
    hexexec_string_free(ptr)
    return s


def check(status: int, err: C.Array | None = None, what: str = ""):
    if status != OK:
        msg = err.value.decode(errors="replace") if err is not None else what
        raise HexexecError(status, msg)


def errbuf(n: int = 1024):
    return C.create_string_buffer(n)
