"""Seeded synthetic pairs for the BASELINE.json configs (input generation only).

Wraps lib/libdreg_synth.so (csrc/synth.cpp); see that file for the recipe.  The
CONFIGS table holds each config's grid (numpy shape (z, y, x)) and solver settings
under SURVEY.md decisions D1-D4 ("A ADMM x B Nesterov" -> max_iters = A*B).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libdreg_synth.so")
_lib = None

# name -> (shape (z,y,x), order n, lambda, theta, warps K, max_iters I, seed, synth config id)
CONFIGS = {
    "config1": dict(shape=(32, 64, 64), order=2, lambda_=0.1, theta=1.0, warps=5, iters=50, seed=1, synth=1),
    "config2": dict(shape=(64, 128, 128), order=2, lambda_=0.1, theta=1.0, warps=7, iters=50, seed=2, synth=2),
    "config3": dict(shape=(64, 128, 128), order=2, lambda_=0.1, theta=1.0, warps=7, iters=50, seed=1000, synth=3),
    "config4": dict(shape=(128, 128, 128), order=3, lambda_=0.05, theta=0.5, warps=15, iters=200, seed=4, synth=4),
    "config5": dict(shape=(192, 256, 256), order=2, lambda_=0.1, theta=1.0, warps=10, iters=50, seed=5, synth=5),
}


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run __graft_entry__.build()")
        _lib = C.CDLL(_LIB)
        F = C.POINTER(C.c_float)
        _lib.dreg_synth_pair.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_int, F, F]
        _lib.dreg_synth_batch.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, F, F, C.c_int]
    return _lib


def make_pair(synth: int, seed: int, shape) -> tuple[np.ndarray, np.ndarray]:
    z, y, x = shape
    f = np.zeros(shape, np.float32)
    m = np.zeros(shape, np.float32)
    F = C.POINTER(C.c_float)
    rc = _load().dreg_synth_pair(synth, seed, x, y, z, f.ctypes.data_as(F), m.ctypes.data_as(F))
    if rc:
        raise ValueError(f"dreg_synth_pair failed ({rc})")
    return f, m


def make_batch(synth: int, seed0: int, n: int, shape, threads: int | None = None,
               out_fixed: np.ndarray | None = None, out_moving: np.ndarray | None = None):
    """n pairs with seeds seed0..seed0+n-1 as [n, z, y, x] arrays (optionally into given buffers)."""
    z, y, x = shape
    f = out_fixed if out_fixed is not None else np.zeros((n,) + tuple(shape), np.float32)
    m = out_moving if out_moving is not None else np.zeros((n,) + tuple(shape), np.float32)
    F = C.POINTER(C.c_float)
    threads = threads or os.cpu_count() or 1
    rc = _load().dreg_synth_batch(synth, seed0, n, x, y, z, f.ctypes.data_as(F), m.ctypes.data_as(F), threads)
    if rc:
        raise ValueError(f"dreg_synth_batch failed ({rc})")
    return f, m


def config_cfg(name: str, order: int | None = None, data_term: int = 2) -> abi.RegCfg:
    """RegistrationConfig for a BASELINE config (levels = 1, tol = 0, log_objective off)."""
    c = CONFIGS[name]
    s = abi.solver_cfg(
        data_term=data_term,
        order=order or c["order"],
        lambda_=c["lambda_"],
        theta=c["theta"],
        max_iters=c["iters"],
        tol=0.0,
        log_objective=False,
    )
    return abi.reg_cfg(s, levels=1, max_warps=(c["warps"],), max_admm_iters=(c["iters"],))
