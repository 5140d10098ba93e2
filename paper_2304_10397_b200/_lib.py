"""ctypes binding of libhpl.so (include/hpl.h, include/hpl_kernels.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no fallback — if libhpl.so is missing or fails to
load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhpl.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -m paper_2304_10397_b200.build` "
        "(there is no CPU fallback)")

lib = ctypes.CDLL(LIB_PATH)

i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
vp = ctypes.c_void_p
ctx_p = ctypes.c_void_p


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


# ---- include/hpl.h
_sig("hpl_init", ctypes.c_int, [i64, i32, i32, i32, u64, ctypes.POINTER(ctx_p)])
_sig("hpl_init_dist", ctypes.c_int, [i64, i32, i32, i32, u64, i32, i32, vp, i32,
                                     ctypes.POINTER(ctx_p)])
_sig("hpl_init_loopback", ctypes.c_int, [i64, i32, i32, i32, u64, i32, vp])
_sig("hpl_get_unique_id", ctypes.c_int, [vp])
_sig("hpl_factor", ctypes.c_int, [ctx_p])
_sig("hpl_solve", ctypes.c_int, [ctx_p, vp])
_sig("hpl_residual", ctypes.c_int, [ctx_p, ctypes.POINTER(ctypes.c_double)])
_sig("hpl_regenerate", ctypes.c_int, [ctx_p])
_sig("hpl_load_local", ctypes.c_int, [ctx_p, vp, i64])
_sig("hpl_load_factor", ctypes.c_int, [ctx_p, vp, i64])
_sig("hpl_local_shape", ctypes.c_int, [ctx_p, ctypes.POINTER(i64), ctypes.POINTER(i64)])
_sig("hpl_free", None, [ctx_p])
_sig("hpl_last_error", ctypes.c_char_p, [ctx_p])
_sig("hpl_singular_column", i64, [ctx_p])
_sig("hpl_get_ipiv", ctypes.c_int, [ctx_p, vp])
_sig("hpl_get_local", ctypes.c_int, [ctx_p, vp, i64])
_sig("hpl_get_timeline", i64, [ctx_p, vp, i64])
_sig("hpl_get_fact_detail", i64, [ctx_p, vp, i64])
_sig("hpl_set_timing", ctypes.c_int, [ctx_p, i32])
_sig("hpl_set_option", ctypes.c_int, [ctx_p, ctypes.c_char_p, i64])
_sig("hpl_launch_count", i64, [ctx_p])
_sig("hpl_last_timing", ctypes.c_int, [ctx_p, vp])
_sig("hpl_phase_stats", ctypes.c_int, [ctx_p, vp])
_sig("hpl_debug_state", ctypes.c_int, [ctx_p, vp, i64])
_sig("hpl_plan_iteration", ctypes.c_int, [i64, i32, i32, i32, i32, i32, i64, vp])
_sig("hpl_plan_fact", ctypes.c_int, [i64, i32, i32, i32, i32, i64, i64, ctypes.c_double, vp])
_sig("hpl_pin_host", ctypes.c_int, [vp, i64, i32])

# ---- include/hpl_kernels.h
_sig("hplk_dgemm_update", ctypes.c_int, [i64, i64, i64, vp, i64, vp, i64, vp, i64, i32])
_sig("hplk_trsm", ctypes.c_int, [i64, i64, vp, i64, vp, i64])
_sig("hplk_panel_fact", ctypes.c_int, [i64, i64, vp, i64, vp, i32, i32, i32, i32,
                                       ctypes.POINTER(i64)])
_sig("hplk_laswp", ctypes.c_int, [i64, i64, vp, i64, i64, i64, vp, i64, i64, vp, i64])
_sig("hplk_back_solve", ctypes.c_int, [i64, i32, vp, i64, vp, vp])
_sig("hplk_rs_exchange", ctypes.c_int, [i64, i64, vp, i64, i32, i32, i64, i64, vp, vp, i64])
_sig("hplk_generate", ctypes.c_int, [u64, i64, i64, i64, i64, i64, vp])
_sig("hplk_residual", ctypes.c_int, [u64, i64, vp, vp, vp, vp, ctypes.POINTER(ctypes.c_double)])
_sig("hplk_dgemm_bench", ctypes.c_int, [i64, i64, i64, i32, i32, vp])
_sig("hplk_dmma_peak", ctypes.c_int, [i32, i32, i32, vp])
_sig("hplk_panel_bench", ctypes.c_int, [i64, i64, i32, i32, i32, vp])

EXPORTED = [
    "hpl_init", "hpl_init_dist", "hpl_init_loopback", "hpl_get_unique_id", "hpl_factor", "hpl_solve",
    "hpl_residual", "hpl_regenerate", "hpl_load_local", "hpl_load_factor", "hpl_local_shape", "hpl_free",
    "hpl_last_error", "hpl_singular_column", "hpl_get_ipiv", "hpl_get_local",
    "hpl_get_timeline", "hpl_get_fact_detail", "hpl_set_timing", "hpl_set_option", "hpl_launch_count",
    "hpl_last_timing", "hpl_phase_stats", "hpl_debug_state", "hpl_plan_iteration", "hpl_plan_fact", "hpl_pin_host",
    "hplk_dgemm_update", "hplk_trsm", "hplk_panel_fact", "hplk_laswp", "hplk_rs_exchange", "hplk_back_solve",
    "hplk_generate", "hplk_residual", "hplk_dgemm_bench", "hplk_dmma_peak", "hplk_panel_bench",
]


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)
