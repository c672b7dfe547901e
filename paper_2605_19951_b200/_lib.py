"""ctypes binding of the C ABI in include/rba_b200.h (libdrba.so, built in-tree).

The product path has no CPU fallback: if the library is missing this module
raises at import time of any GPU entry point (``load()``), loudly.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = ["load", "check", "RbaError", "LIB_PATH", "ptr"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdrba.so")

RBA_OK, RBA_ERR_INVALID, RBA_ERR_CUDA, RBA_ERR_SOLVE, RBA_ERR_CACHE_MISS, RBA_ERR_STATE, \
    RBA_ERR_OOM = range(7)


class RbaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None

i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
vp = C.c_void_p

_SIGS = {
    "rba_last_error": (C.c_char_p, []),
    "rba_version": (C.c_int, []),
    "rba_symbolic_analyze": (C.c_int, [i64, vp, vp, vp, i32, C.POINTER(vp)]),
    "rba_symbolic_stats": (C.c_int, [vp, vp, vp]),
    "rba_symbolic_array": (C.c_int, [vp, C.c_char_p, vp, i64, C.POINTER(i64)]),
    "rba_symbolic_destroy": (None, [vp]),
    "rba_mesh_prepare": (C.c_int, [i64, i64, i32, vp, vp, vp, vp, vp, vp, i32, vp]),
    "rba_ctx_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "rba_ctx_destroy": (None, [vp]),
    "rba_set_mesh": (C.c_int, [vp, i64, i64, i32, vp, vp, vp, vp, vp, vp, i32]),
    "rba_set_observation": (C.c_int, [vp, i64, vp, vp, vp]),
    "rba_set_sources": (C.c_int, [vp, i32, vp]),
    "rba_set_sources_complex": (C.c_int, [vp, i32, vp]),
    "rba_set_poles": (C.c_int, [vp, i32, vp, i32, vp, i32, vp]),
    "rba_set_model": (C.c_int, [vp, vp]),
    "rba_set_model_d": (C.c_int, [vp, vp]),
    "rba_factor": (C.c_int, [vp]),
    "rba_factor_values": (C.c_int, [vp, i32, vp]),
    "rba_pattern": (C.c_int, [vp, C.POINTER(i64), vp, vp, vp, vp]),
    "rba_solve": (C.c_int, [vp, i32, vp, vp, i32, i32]),
    "rba_solve_d": (C.c_int, [vp, i32, vp, vp, i32, i32]),
    "rba_forward_partial": (C.c_int, [vp, vp]),
    "rba_get_g": (C.c_int, [vp, i32, vp]),
    "rba_get_factor": (C.c_int, [vp, i32, vp, i64]),
    "rba_jvp_partial": (C.c_int, [vp, vp, vp]),
    "rba_vjp_partial": (C.c_int, [vp, vp, vp]),
    "rba_combine_data": (C.c_int, [vp, vp, vp, i32, vp]),
    "rba_combine_cells": (C.c_int, [vp, vp, vp, vp]),
    "rba_set_reg": (C.c_int, [vp, i64, vp, vp, vp]),
    "rba_reg_apply": (C.c_int, [vp, i32, vp, f64, vp, i32]),
    "rba_vec_axpby": (C.c_int, [vp, i64, f64, vp, f64, vp, vp]),
    "rba_vec_mul": (C.c_int, [vp, i64, vp, vp, f64, vp]),
    "rba_vec_dot": (C.c_int, [vp, i64, vp, vp, vp]),
    "rba_vec_lsqr_xw": (C.c_int, [vp, i64, f64, f64, vp, vp, vp, vp]),
    "rba_info": (C.c_int, [vp, vp]),
    "rba_memory": (C.c_int, [vp, vp]),
    "rba_sync": (C.c_int, [vp]),
    "rba_timings": (C.c_int, [vp, vp]),
    "rba_set_timing": (C.c_int, [vp, i32]),
    "rba_timings_detail": (C.c_int, [vp, vp]),
    "rba_get_g_d": (C.c_int, [vp, i32, vp]),
    "rba_set_g": (C.c_int, [vp, i32, vp]),
    "rba_factor_stats": (C.c_int, [vp, i32, vp]),
    "rba_set_option": (C.c_int, [vp, C.c_char_p, i64]),
    "rba_set_reg_L": (C.c_int, [vp, i64, vp, vp, vp]),
    "rba_oz_stats": (C.c_int, [vp, vp]),
    "rba_oz_prof": (C.c_int, [vp, vp, C.c_int]),
    "rba_box_generate": (C.c_int, [i32, f64, vp, C.POINTER(vp)]),
    "rba_box_info": (C.c_int, [vp, vp]),
    "rba_box_get": (C.c_int, [vp, C.c_char_p, vp, i64]),
    "rba_box_destroy": (None, [vp]),
    "rba_box_last_error": (C.c_char_p, []),
    "rba_spectral_bound": (C.c_int, [i64, vp, vp, vp, vp]),
    "rba_reg_L_apply": (C.c_int, [vp, vp, f64, vp, i32]),
}

EXPORTED = tuple(_SIGS)


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'` "
                          "(no CPU fallback exists for the shifted-solve path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a) -> int | None:
    """Host pointer of a C-contiguous numpy array, or device pointer of a torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    return a.data_ptr()


def check(rc: int):
    if rc == RBA_OK:
        return
    msg = load().rba_last_error().decode(errors="replace")
    from .shifted import CacheMissError, SolveError  # avoid cycle at import time
    if rc == RBA_ERR_SOLVE:
        raise SolveError(msg)
    if rc == RBA_ERR_CACHE_MISS:
        raise CacheMissError(msg)
    if rc == RBA_ERR_INVALID:
        raise ValueError(msg)
    if rc == RBA_ERR_OOM:
        raise MemoryError(msg)
    raise RbaError(rc, msg)
