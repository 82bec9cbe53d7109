"""ctypes loader for the compiled C oracle (oracle/liboracle.so).  TEST INFRASTRUCTURE."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

CFLAGS = ["-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain IEEE double, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        d, i, i64, u64 = C.c_double, C.c_int, C.c_int64, C.c_uint64
        p = C.c_void_p
        L.orc_glass_index.restype = d
        L.orc_glass_index.argtypes = [i, p, d]
        L.orc_trace.restype = None
        L.orc_trace.argtypes = [p, i, p, u64, i64, p, p, d, p, p, p, p, p, p, p, p]
        L.orc_mlp_forward.restype = None
        L.orc_mlp_forward.argtypes = [i, p, p, p, i64, p, p]
        L.orc_map_eval.restype = None
        L.orc_map_eval.argtypes = [i, p, p, p, i, p, p, p, p, i64, p, p, p, p, p, p, p, p, p]
        L.orc_splat.restype = i64
        L.orc_splat.argtypes = [i, i, i, d, d, d, d, p, i64, p, p, p, p, p, p, C.c_float]
        L.orc_shade_plane.restype = None
        L.orc_shade_plane.argtypes = [d, d, d, d, i, i64, C.c_float, p, i64, p, p, p, p, p, p, p, p]
        L.orc_shade_cards.restype = None
        L.orc_shade_cards.argtypes = [p, i, d, d, i, i64, C.c_float, p, i64, p, p, p, p, p, p, p, p]
        _lib = L
    return _lib


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def glass_index(model: int, coeffs, lam_nm: float) -> float:
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    return float(lib().orc_glass_index(int(model), ptr(c), float(lam_nm)))
