"""ctypes binding of oracle/checker_wide.c: checker.py's exact definitions
(Eq.1 value, bisection + (n+1)-bit midpoint rounding) with exact 768-bit
integer comparisons instead of Fractions -- fast enough for S:443's 1e7
random pairs.  TEST INFRASTRUCTURE ONLY; shares no code with posit_oracle.c
or the CUDA path."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "checker_wide.c")
_LIB = os.path.join(_HERE, "libchecker_wide.so")
_lock = threading.Lock()
_lib = None
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", "-o", _LIB, _SRC], check=True)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
            L.cw_op1.argtypes = [i32, u64, u64, i32, i32]
            L.cw_op1.restype = u64
            L.cw_check.argtypes = [i32, vp, vp, vp, vp, i64, i32, i32]
            L.cw_check.restype = i64
            L.cw_threads.restype = i32
            _lib = L
    return _lib


def op1(op: str, a: int, b: int = 0, n: int = 32, es: int = 2) -> int:
    return int(lib().cw_op1(OPS[op], a, b, n, es))


def expected(op: str, a, b=None, got=None, n: int = 32, es: int = 2):
    """-> (want array, number of positions where want != got)."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = None if b is None else np.ascontiguousarray(b, dtype=np.uint32)
    got = np.zeros_like(a) if got is None else np.ascontiguousarray(got, dtype=np.uint32)
    want = np.empty_like(a)
    nbad = lib().cw_check(OPS[op], a.ctypes.data, None if b is None else b.ctypes.data, got.ctypes.data,
                          want.ctypes.data, a.size, n, es)
    return want, int(nbad)
