"""Exactly rounded element-wise fma for the CPU oracle — TEST INFRASTRUCTURE.

``fma(a, b, c)`` broadcasts like NumPy and returns RN(a*b + c) with a single
rounding, computed by C99 ``fma()`` (oracle/native/fma_arr.c, glibc: correctly
rounded). The shared object is built on first use with gcc into
oracle/native/libfma_arr.so (``__graft_entry__.build()`` also builds it).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native")
SRC = os.path.join(_HERE, "fma_arr.c")
LIB = os.path.join(_HERE, "libfma_arr.so")
_lock = threading.Lock()
_lib = None


def build() -> str:
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", LIB, SRC, "-lm"], check=True)
    return LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
                build()
            lib = ctypes.CDLL(LIB)
            p = ctypes.c_void_p
            lib.fma_arr.argtypes = [p, p, p, p, ctypes.c_long]
            lib.fma_arr.restype = None
            _lib = lib
    return _lib


def fma(a, b, c) -> np.ndarray:
    lib = _load()
    a, b, c = np.broadcast_arrays(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64),
                                  np.asarray(c, dtype=np.float64))
    a, b, c = (np.ascontiguousarray(x) for x in (a, b, c))
    out = np.empty(a.shape, dtype=np.float64)
    if out.size:
        lib.fma_arr(a.ctypes.data, b.ctypes.data, c.ctypes.data, out.ctypes.data, out.size)
    return out
