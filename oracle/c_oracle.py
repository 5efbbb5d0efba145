"""ctypes binding of the C restatement ``oracle/sw_oracle.c`` -- TEST
INFRASTRUCTURE ONLY (tests, smoke() checker, bench CPU baseline)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libsw_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        for suf, ct in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            fn = getattr(L, f"sw_oracle_step_{suf}")
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 6 + \
                [ct] * 4 + [ctypes.c_int, ctypes.c_int]
            fb = getattr(L, f"sw_oracle_boundary_{suf}")
            fb.restype = ctypes.c_int
            fb.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [ctypes.c_void_p] * 3 + [ctypes.c_int]
        L.sw_oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


BC = {"reflective": 0, "periodic": 1}


def _suf(a):
    return {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64"}[a.dtype]


def max_threads() -> int:
    return lib().sw_oracle_max_threads()


def step(H, U, V, dx, dy, dt, g=9.8, boundary="reflective", out=None, threads=None):
    """One oracle step (DSL op order) + boundary fill of the outputs."""
    for a in (H, U, V):
        assert a.flags.c_contiguous and a.dtype == H.dtype
    ny2, nx2 = H.shape
    if out is None:
        out = (np.empty_like(H), np.empty_like(U), np.empty_like(V))
    oH, oU, oV = out
    fn = getattr(lib(), f"sw_oracle_step_{_suf(H)}")
    rc = fn(nx2 - 2, ny2 - 2, nx2, H.ctypes.data, U.ctypes.data, V.ctypes.data,
            oH.ctypes.data, oU.ctypes.data, oV.ctypes.data, dx, dy, dt, g,
            BC[boundary], threads or max_threads())
    if rc:
        raise RuntimeError(f"sw_oracle_step rc={rc}")
    return oH, oU, oV


def apply_boundary(H, U, V, boundary="reflective"):
    ny2, nx2 = H.shape
    fn = getattr(lib(), f"sw_oracle_boundary_{_suf(H)}")
    fn(nx2 - 2, ny2 - 2, nx2, H.ctypes.data, U.ctypes.data, V.ctypes.data, BC[boundary])
    return H, U, V


def run_fixed(H, U, V, steps, dx, dy, dt, g=9.8, boundary="reflective", threads=None):
    """``steps`` double-buffered steps at fixed dt; returns the final state."""
    a = (H.copy(), U.copy(), V.copy())
    b = (np.empty_like(H), np.empty_like(U), np.empty_like(V))
    for _ in range(steps):
        step(*a, dx, dy, dt, g, boundary, out=b, threads=threads)
        a, b = b, a
    return a
