"""ctypes binding of the CPU oracle (oracle/posit_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product path
(paper_2401_14117_b200) never imports this module.

Every function here is argument marshalling; the arithmetic is in
posit_oracle.c, whose header cites the PAPER.md passages each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "posit_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

P32_ONE = 0x40000000
P32_MONE = 0xC0000000
P32_NAR = 0x80000000


def build(force: bool = False) -> str:
    """Compile posit_oracle.c into oracle/liboracle.so (plain gcc -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            u32, i32, i64, dbl = ctypes.c_uint32, ctypes.c_int, ctypes.c_int64, ctypes.c_double
            vp = ctypes.c_void_p
            for name in ("or_add", "or_sub", "or_mul", "or_div"):
                getattr(L, name).argtypes = [u32, u32, i32, i32]
                getattr(L, name).restype = u32
            for name in ("or_sqrt", "or_neg"):
                getattr(L, name).argtypes = [u32, i32, i32]
                getattr(L, name).restype = u32
            L.or_from_f64.argtypes = [dbl, i32, i32]
            L.or_from_f64.restype = u32
            L.or_to_f64.argtypes = [u32, i32, i32]
            L.or_to_f64.restype = dbl
            L.or_fraction_bits.argtypes = [u32, i32, i32]
            L.or_fraction_bits.restype = i32
            L.or_scale.argtypes = [u32, i32, i32]
            L.or_scale.restype = i32
            L.or_num_threads.argtypes = []
            L.or_num_threads.restype = i32
            L.or_from_f64_array.argtypes = [vp, vp, i64, i32, i32]
            L.or_to_f64_array.argtypes = [vp, vp, i64, i32, i32]
            L.or_vec_op.argtypes = [i32, vp, vp, vp, i64, i32, i32]
            L.or_roundtrip_all32.argtypes = [ctypes.POINTER(ctypes.c_int64)]
            L.or_roundtrip_all32.restype = ctypes.c_int64
            L.or_gemm.argtypes = [ctypes.c_char, ctypes.c_char, i64, i64, i64, u32, vp, i64, vp, i64, u32, vp, i64]
            L.or_gemm.restype = i32
            L.or_gemm_eq2.argtypes = [ctypes.c_char, ctypes.c_char, i64, i64, i64, u32, vp, i64, vp, i64, u32, vp, i64]
            L.or_gemm_eq2.restype = i32
            L.or_syrk_lower.argtypes = [i64, i64, u32, vp, i64, u32, vp, i64]
            L.or_syrk_lower.restype = i32
            L.or_trsm_llnu.argtypes = [i64, i64, vp, i64, vp, i64]
            L.or_trsm_llnu.restype = i32
            L.or_trsm_rltn.argtypes = [i64, i64, vp, i64, vp, i64]
            L.or_trsm_rltn.restype = i32
            L.or_getrf.argtypes = [i64, i64, vp, i64, vp, vp]
            L.or_getrf.restype = i32
            L.or_getrf_steps.argtypes = [i64, i64, vp, i64, vp, vp, i64, i64]
            L.or_getrf_steps.restype = i32
            L.or_potrf_lower.argtypes = [i64, vp, i64, vp]
            L.or_potrf_lower.restype = i32
            L.or_getrs.argtypes = [i64, vp, i64, vp, vp]
            L.or_getrs.restype = i32
            L.or_potrs_lower.argtypes = [i64, vp, i64, vp]
            L.or_potrs_lower.restype = i32
            _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


# ---- scalar ops on patterns (n, es generic; default Posit(32,2)) -------------
def add(a, b, n=32, es=2): return lib().or_add(a, b, n, es)
def sub(a, b, n=32, es=2): return lib().or_sub(a, b, n, es)
def mul(a, b, n=32, es=2): return lib().or_mul(a, b, n, es)
def div(a, b, n=32, es=2): return lib().or_div(a, b, n, es)
def sqrt(a, n=32, es=2): return lib().or_sqrt(a, n, es)
def neg(a, n=32, es=2): return lib().or_neg(a, n, es)
def from_f64(x, n=32, es=2): return lib().or_from_f64(float(x), n, es)
def to_f64(a, n=32, es=2): return lib().or_to_f64(a, n, es)
def fraction_bits(a, n=32, es=2): return lib().or_fraction_bits(a, n, es)
def scale(a, n=32, es=2): return lib().or_scale(a, n, es)
def num_threads() -> int: return lib().or_num_threads()


_OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4, "neg": 5}


def vec_op(op: str, a, b=None, n=32, es=2) -> np.ndarray:
    a = _u32(a)
    b = a if b is None else _u32(b)
    out = np.empty_like(a)
    lib().or_vec_op(_OPS[op], _ptr(a), _ptr(b), _ptr(out), a.size, n, es)
    return out


def from_f64_array(x, n=32, es=2) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty(x.shape, dtype=np.uint32)
    lib().or_from_f64_array(_ptr(x), _ptr(out), x.size, n, es)
    return out


def to_f64_array(p, n=32, es=2) -> np.ndarray:
    p = _u32(p)
    out = np.empty(p.shape, dtype=np.float64)
    lib().or_to_f64_array(_ptr(p), _ptr(out), p.size, n, es)
    return out


def roundtrip_all32() -> tuple[int, int]:
    viol = ctypes.c_int64(0)
    bad = lib().or_roundtrip_all32(ctypes.byref(viol))
    return int(bad), int(viol.value)


# ---- linear algebra (Posit(32,2), row-major, order contract) ------------------
def gemm(A, B, C=None, transa="N", transb="N", alpha=P32_MONE, beta=P32_ONE) -> np.ndarray:
    """Returns op-updated copy of C (C <- beta*C (+/-) op(A) op(B))."""
    A, B = _u32(A), _u32(B)
    m = A.shape[0] if transa == "N" else A.shape[1]
    k = A.shape[1] if transa == "N" else A.shape[0]
    n = B.shape[1] if transb == "N" else B.shape[0]
    C = np.zeros((m, n), np.uint32) if C is None else _u32(C).copy()
    rc = lib().or_gemm(transa.encode(), transb.encode(), m, n, k, alpha, _ptr(A), A.shape[1],
                       _ptr(B), B.shape[1], beta, _ptr(C), max(n, 1))
    if rc != 0:
        raise ValueError(f"or_gemm returned {rc}")
    return C


def gemm_eq2(A, B, C, alpha, beta, transa="N", transb="N") -> np.ndarray:
    """Eq.2 in SPEC S:200's order: t = sum of products from 0, then (alpha t) + (beta C)."""
    A, B = _u32(A), _u32(B)
    m = A.shape[0] if transa == "N" else A.shape[1]
    k = A.shape[1] if transa == "N" else A.shape[0]
    n = B.shape[1] if transb == "N" else B.shape[0]
    C = _u32(C).copy()
    rc = lib().or_gemm_eq2(transa.encode(), transb.encode(), m, n, k, alpha, _ptr(A), A.shape[1],
                           _ptr(B), B.shape[1], beta, _ptr(C), max(n, 1))
    if rc != 0:
        raise ValueError(f"or_gemm_eq2 returned {rc}")
    return C


def syrk_lower(A, C, alpha=P32_MONE, beta=P32_ONE) -> np.ndarray:
    A = _u32(A)
    C = _u32(C).copy()
    rc = lib().or_syrk_lower(A.shape[0], A.shape[1], alpha, _ptr(A), A.shape[1], beta, _ptr(C), C.shape[1])
    if rc != 0:
        raise ValueError(f"or_syrk_lower returned {rc}")
    return C


def trsm_llnu(L, B) -> np.ndarray:
    L, B = _u32(L), _u32(B).copy()
    lib().or_trsm_llnu(B.shape[0], B.shape[1], _ptr(L), L.shape[1], _ptr(B), B.shape[1])
    return B


def trsm_rltn(L, B) -> np.ndarray:
    L, B = _u32(L), _u32(B).copy()
    lib().or_trsm_rltn(B.shape[0], B.shape[1], _ptr(L), L.shape[1], _ptr(B), B.shape[1])
    return B


def getrf(A) -> tuple[np.ndarray, np.ndarray, int]:
    A = _u32(A).copy()
    m, n = A.shape
    ipiv = np.zeros(min(m, n), np.int32)
    info = np.zeros(1, np.int32)
    lib().or_getrf(m, n, _ptr(A), n, _ptr(ipiv), _ptr(info))
    return A, ipiv, int(info[0])


def getrf_steps(A, ipiv, info, k0: int, k1: int) -> None:
    """Steps k0 <= k < k1 of the textbook LU in place on A (uint32, C-contiguous),
    ipiv (int32) and info (int32 array of 1): resumable form of getrf."""
    assert A.flags.c_contiguous and A.dtype == np.uint32 and ipiv.dtype == np.int32 and info.dtype == np.int32
    m, n = A.shape
    rc = lib().or_getrf_steps(m, n, _ptr(A), n, _ptr(ipiv), _ptr(info), k0, k1)
    if rc != 0:
        raise ValueError(f"or_getrf_steps returned {rc}")


def potrf_lower(A) -> tuple[np.ndarray, int]:
    A = _u32(A).copy()
    n = A.shape[0]
    info = np.zeros(1, np.int32)
    lib().or_potrf_lower(n, _ptr(A), n, _ptr(info))
    return A, int(info[0])


def getrs(LU, ipiv, b) -> np.ndarray:
    LU, b = _u32(LU), _u32(b).copy()
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int32)
    lib().or_getrs(LU.shape[0], _ptr(LU), LU.shape[1], _ptr(ipiv), _ptr(b))
    return b


def potrs_lower(L, b) -> np.ndarray:
    L, b = _u32(L), _u32(b).copy()
    lib().or_potrs_lower(L.shape[0], _ptr(L), L.shape[1], _ptr(b))
    return b
