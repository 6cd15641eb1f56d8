"""Loader for the C depth renderer (input generation only)."""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "render.c")
_LIB = os.path.join(_HERE, "librender.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            L.synth_render.argtypes = [ctypes.c_int32, ctypes.c_int32, dp, dp, dp,
                                       ctypes.c_int32, dp, ctypes.c_int32, dp, ctypes.c_int32, dp, dp]
            L.synth_render.restype = None
            _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def render(W, H, K, R, C, rects, boxes, obbs):
    K = np.ascontiguousarray(K, dtype=np.float64)
    R = np.ascontiguousarray(R, dtype=np.float64).reshape(9)
    C = np.ascontiguousarray(C, dtype=np.float64)
    rects = np.ascontiguousarray(np.asarray(rects, dtype=np.float64).reshape(-1, 6))
    boxes = np.ascontiguousarray(np.asarray(boxes, dtype=np.float64).reshape(-1, 6))
    obbs = np.ascontiguousarray(np.asarray(obbs, dtype=np.float64).reshape(-1, 7))
    out = np.empty(W * H, dtype=np.float64)
    lib().synth_render(W, H, _dp(K), _dp(R), _dp(C), len(rects), _dp(rects), len(boxes), _dp(boxes),
                       len(obbs), _dp(obbs), _dp(out))
    return out
