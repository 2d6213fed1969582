"""ctypes wrapper of oracle/band_inertia.c — TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libband_inertia.so")
_lib = None


def build():
    os.makedirs(os.path.dirname(_SO), exist_ok=True)
    src = os.path.join(_HERE, "band_inertia.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _SO, src])
    return _SO


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.band_inertia_count.restype = ctypes.c_long
        _lib.band_inertia_count.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_int, ctypes.c_long, ctypes.c_double]
    return _lib


def count_below(ab_lower, bb_lower, sigma):
    """#eigenvalues of the band pencil below sigma ('L' band storage)."""
    ab = np.ascontiguousarray(ab_lower, dtype=np.float64)
    bb = None if bb_lower is None else np.ascontiguousarray(bb_lower, dtype=np.float64)
    n = ab.shape[1]
    r = _load().band_inertia_count(ab.ctypes.data, ab.shape[0] - 1,
                                   None if bb is None else bb.ctypes.data,
                                   0 if bb is None else bb.shape[0] - 1, n, float(sigma))
    if r < 0:
        raise MemoryError
    return int(r)
