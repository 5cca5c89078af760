"""paper_2401_14117_b200 -- Posit(32,2) LU / Cholesky hot path on NVIDIA B200.

Thin Python binding of the C ABI in ``include/posit_b200.h``
(``libposit_b200.so``, built in-tree by ``paper_2401_14117_b200.build``).
Every function here only marshals arguments -- torch tensors (uint32 patterns
stored as int32, device memory) become raw pointers, the current torch CUDA
stream becomes the ``cudaStream_t`` -- and calls the library of the same
name.  All arithmetic runs in the CUDA kernels.  There is no CPU fallback:
if the library or a CUDA device is missing, the calls raise.

Posit patterns live in ``torch.int32`` tensors (torch has no uint32 arithmetic
on CUDA); the bits are the Posit(32,2) encoding (0x40000000 = 1.0).
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "lib", "PositError", "posit_gemm", "posit_gemm_eq2", "posit_gemm_naive", "posit_gemm_host", "posit_syrk", "posit_trsm",
    "posit_getrf", "posit_getrf_panel", "posit_getrs", "posit_potrs", "posit_laswp", "posit_potrf", "posit_from_f64", "posit_to_f64",
    "posit_vec_op", "posit_vec_dmac", "posit_iamax_key", "posit_kernel_launches", "POSIT_ONE", "POSIT_MONE", "POSIT_NAR", "OPS",
]

POSIT_ONE = 0x40000000
POSIT_MONE = 0xC0000000
POSIT_NAR = 0x80000000
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4, "dadd": 5, "dmul": 6, "ddiv": 8, "dsqrt": 9}

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POSIT_LIB_PATH") or os.path.join(_HERE, "libposit_b200.so")
_lib = None


class PositError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load libposit_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PositError(f"{LIB_PATH} missing: run `python -m paper_2401_14117_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        c_char, i64, u32, vp, sz = ctypes.c_char, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t
        gemm_args = [c_char, c_char, i64, i64, i64, u32, vp, i64, vp, i64, u32, vp, i64, vp]
        L.posit_gemm.argtypes = gemm_args
        L.posit_gemm_naive.argtypes = gemm_args
        L.posit_gemm_host.argtypes = gemm_args[:-1] + [vp, sz, vp]
        L.posit_gemm_eq2.argtypes = gemm_args[:-1] + [vp, sz, vp]
        L.posit_gemm_eq2_work_bytes.argtypes = [i64, i64]
        L.posit_gemm_eq2_work_bytes.restype = sz
        L.posit_gemm_host_work_bytes.argtypes = [i64, i64, i64]
        L.posit_gemm_host_work_bytes.restype = sz
        L.posit_syrk.argtypes = [c_char, c_char, i64, i64, u32, vp, i64, u32, vp, i64, vp]
        L.posit_trsm.argtypes = [c_char, c_char, c_char, c_char, i64, i64, u32, vp, i64, vp, i64, vp]
        L.posit_getrf.argtypes = [i64, i64, vp, i64, vp, vp, i64, vp, sz, vp]
        L.posit_getrf_work_bytes.argtypes = [i64, i64, i64]
        L.posit_getrf_work_bytes.restype = sz
        L.posit_getrf_panel.argtypes = [i64, i64, vp, i64, vp, vp, i64, vp, sz, vp]
        L.posit_laswp.argtypes = [i64, vp, i64, i64, i64, vp, i64, vp]
        L.posit_potrf.argtypes = [c_char, i64, vp, i64, vp, i64, vp, sz, vp]
        L.posit_potrf_work_bytes.argtypes = [i64, i64]
        L.posit_potrf_work_bytes.restype = sz
        L.posit_getrs.argtypes = [c_char, i64, vp, i64, vp, vp, vp]
        L.posit_potrs.argtypes = [c_char, i64, vp, i64, vp, vp]
        L.posit_iamax_key.argtypes = [i64, vp, i64, vp, i64, vp, vp]
        L.posit_from_f64.argtypes = [vp, vp, i64, vp]
        L.posit_to_f64.argtypes = [vp, vp, i64, vp]
        L.posit_vec_op.argtypes = [ctypes.c_int, vp, vp, vp, i64, vp]
        L.posit_vec_dmac.argtypes = [vp, vp, vp, vp, i64, vp]
        L.posit_kernel_launches.restype = ctypes.c_uint64
        L.posit_strerror.argtypes = [ctypes.c_int]
        L.posit_strerror.restype = ctypes.c_char_p
        L.posit_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def posit_kernel_launches() -> int:
    """Kernels launched by libposit_b200 in this process so far."""
    return int(lib().posit_kernel_launches())


def _check(rc: int, name: str) -> None:
    if rc != 0:
        L = lib()
        raise PositError(f"{name} returned {rc}: {L.posit_strerror(rc).decode()} {L.posit_last_error().decode()}")


def _ptr(t) -> int:
    if t is None:
        return 0
    if not t.is_cuda:
        raise PositError("expected a CUDA tensor (device memory)")
    return t.data_ptr()


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ld(t) -> int:
    return t.stride(0) if t.dim() == 2 else max(t.shape[-1], 1)


# ---- argument checks (the C ABI takes raw pointers; a wrong dtype, device or
# layout would silently read the wrong words or run out of bounds) ------------
def _mat(t, name: str, host: bool = False):
    """A row-major int32 pattern matrix (a view with a row stride is fine; the
    elements of a row must be contiguous).  Returns (rows, cols)."""
    import torch
    if t.dtype != torch.int32:
        raise PositError(f"{name}: expected torch.int32 posit patterns, got {t.dtype}")
    if t.dim() != 2:
        raise PositError(f"{name}: expected a 2-D matrix, got shape {tuple(t.shape)}")
    if host == t.is_cuda:
        raise PositError(f"{name}: expected a {'host' if host else 'CUDA'} tensor")
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise PositError(f"{name}: row elements must be contiguous (stride(1) == 1), got strides {t.stride()}")
    if t.shape[0] > 1 and t.stride(0) < max(t.shape[1], 1):
        raise PositError(f"{name}: row stride {t.stride(0)} < {t.shape[1]} columns")
    return t.shape[0], t.shape[1]


def _vec(t, name: str, dtype, min_len: int):
    """A contiguous device vector of at least min_len elements of dtype."""
    if t.dtype != dtype:
        raise PositError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise PositError(f"{name}: expected a CUDA tensor")
    if not t.is_contiguous():
        raise PositError(f"{name}: expected a contiguous tensor")
    if t.numel() < min_len:
        raise PositError(f"{name}: needs at least {min_len} elements, has {t.numel()}")


def _gemm_shapes(A, B, C, transa: str, transb: str, host: bool = False):
    if transa not in ("N", "T") or transb not in ("N", "T"):
        raise PositError(f"transa/transb must be 'N' or 'T', got {transa!r}/{transb!r}")
    ar, ac = _mat(A, "A", host)
    br, bc = _mat(B, "B", host)
    m, n = _mat(C, "C", host)
    am, k = (ar, ac) if transa == "N" else (ac, ar)
    bk, bn = (br, bc) if transb == "N" else (bc, br)
    if am != m or bn != n or bk != k:
        raise PositError(f"op(A) {am}x{k}, op(B) {bk}x{bn} and C {m}x{n} do not conform")
    return m, n, k


def posit_gemm(A, B, C, transb: str = "N", alpha: int = POSIT_MONE, beta: int = POSIT_ONE, stream=None,
               transa: str = "N") -> None:
    """C <- alpha*op(A)*op(B) + beta*C in place (row-major int32 pattern tensors; views with row stride allowed)."""
    m, n, k = _gemm_shapes(A, B, C, transa, transb)
    _check(lib().posit_gemm(transa.encode(), transb.encode(), m, n, k, alpha, _ptr(A), _ld(A), _ptr(B), _ld(B), beta,
                            _ptr(C), _ld(C), _stream(stream)), "posit_gemm")


def posit_gemm_eq2(A, B, C, alpha: int, beta: int, transb: str = "N", transa: str = "N", stream=None,
                   work=None) -> None:
    """Eq.2 for any alpha, beta (posit patterns) in SPEC S:200's order: t = sum of products, then
    C <- alpha t + beta C (see include/posit_b200.h)."""
    m, n, k = _gemm_shapes(A, B, C, transa, transb)
    w, wb = _work(int(lib().posit_gemm_eq2_work_bytes(m, n)), C, work)
    _check(lib().posit_gemm_eq2(transa.encode(), transb.encode(), m, n, k, alpha, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                beta, _ptr(C), _ld(C), _ptr(w), wb, _stream(stream)), "posit_gemm_eq2")


def posit_gemm_naive(A, B, C, transb: str = "N", alpha: int = POSIT_MONE, beta: int = POSIT_ONE, stream=None,
                     transa: str = "N") -> None:
    m, n, k = _gemm_shapes(A, B, C, transa, transb)
    _check(lib().posit_gemm_naive(transa.encode(), transb.encode(), m, n, k, alpha, _ptr(A), _ld(A), _ptr(B), _ld(B), beta,
                                  _ptr(C), _ld(C), _stream(stream)), "posit_gemm_naive")


def posit_gemm_host(A, B, C, dwork, transb: str = "N", alpha: int = POSIT_MONE, beta: int = POSIT_ONE,
                    stream=None, transa: str = "N") -> None:
    """HOST-buffer GEMM: A, B, C are CPU (pinned) int32 tensors; dwork a CUDA byte workspace."""
    m, n, k = _gemm_shapes(A, B, C, transa, transb, host=True)
    for t in (A, B, C):
        if not t.is_contiguous():
            raise PositError("posit_gemm_host expects contiguous host tensors")
    if not dwork.is_cuda or dwork.numel() * dwork.element_size() < posit_gemm_host_work_bytes(m, n, k):
        raise PositError("posit_gemm_host: dwork must be a CUDA tensor of posit_gemm_host_work_bytes() bytes")
    _check(lib().posit_gemm_host(transa.encode(), transb.encode(), m, n, k, alpha, A.data_ptr(), _ld(A), B.data_ptr(), _ld(B),
                                 beta, C.data_ptr(), _ld(C), _ptr(dwork), dwork.numel() * dwork.element_size(),
                                 _stream(stream)), "posit_gemm_host")


def posit_gemm_host_work_bytes(m: int, n: int, k: int) -> int:
    return int(lib().posit_gemm_host_work_bytes(m, n, k))


def posit_syrk(A, C, alpha: int = POSIT_MONE, beta: int = POSIT_ONE, stream=None) -> None:
    """Lower triangle of C <- alpha*A*A^T + beta*C."""
    n, k = _mat(A, "A")
    if _mat(C, "C") != (n, n):
        raise PositError(f"C must be {n}x{n}, got {tuple(C.shape)}")
    _check(lib().posit_syrk(b"L", b"N", n, k, alpha, _ptr(A), _ld(A), beta, _ptr(C), _ld(C), _stream(stream)),
           "posit_syrk")


def posit_trsm(side: str, uplo: str, transa: str, diag: str, A, B, stream=None) -> None:
    m, n = _mat(B, "B")
    na = m if side == "L" else n
    if _mat(A, "A")[0] < na or A.shape[1] < na:
        raise PositError(f"A must be at least {na}x{na} for side {side!r}, got {tuple(A.shape)}")
    _check(lib().posit_trsm(side.encode(), uplo.encode(), transa.encode(), diag.encode(), m, n, POSIT_ONE, _ptr(A),
                            _ld(A), _ptr(B), _ld(B), _stream(stream)), "posit_trsm")


def _work(nbytes: int, like, work):
    import torch
    if work is None:
        work = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=like.device)
    return work, work.numel() * work.element_size()


def posit_getrf(A, ipiv, info, nb: int = 256, stream=None, work=None) -> None:
    """In-place blocked LU with partial pivoting; ipiv (int32, min(m,n)) and info (int32, 1) are device tensors.
    work: optional device byte tensor of posit_getrf_work_bytes() bytes (allocated here if None)."""
    import torch
    m, n = _mat(A, "A")
    _vec(ipiv, "ipiv", torch.int32, min(m, n))
    _vec(info, "info", torch.int32, 1)
    w, wb = _work(int(lib().posit_getrf_work_bytes(m, n, nb)), A, work)
    _check(lib().posit_getrf(m, n, _ptr(A), _ld(A), _ptr(ipiv), _ptr(info), nb, _ptr(w), wb, _stream(stream)),
           "posit_getrf")


def posit_getrf_panel(P, ipiv, info, row_base: int = 0, stream=None, work=None) -> None:
    import torch
    m, b = _mat(P, "P")
    _vec(ipiv, "ipiv", torch.int32, min(m, b))
    _vec(info, "info", torch.int32, 1)
    w, wb = _work(int(lib().posit_getrf_work_bytes(m, b, b)), P, work)
    _check(lib().posit_getrf_panel(m, b, _ptr(P), _ld(P), _ptr(ipiv), _ptr(info), row_base, _ptr(w), wb,
                                   _stream(stream)), "posit_getrf_panel")


def posit_laswp(A, k1: int, k2: int, ipiv, ipiv_base: int = 0, stream=None) -> None:
    import torch
    rows, ncols = _mat(A, "A")
    if not (0 <= k1 <= k2 <= rows):
        raise PositError(f"laswp rows [{k1}, {k2}) outside the {rows} rows of A")
    _vec(ipiv, "ipiv", torch.int32, k2)
    _check(lib().posit_laswp(ncols, _ptr(A), _ld(A), k1, k2, _ptr(ipiv), ipiv_base, _stream(stream)), "posit_laswp")


def posit_potrf(A, info, nb: int = 256, stream=None) -> None:
    import torch
    n, n2 = _mat(A, "A")
    if n2 != n:
        raise PositError(f"posit_potrf needs a square matrix, got {tuple(A.shape)}")
    _vec(info, "info", torch.int32, 1)
    _check(lib().posit_potrf(b"L", n, _ptr(A), _ld(A), _ptr(info), nb, None, 0, _stream(stream)), "posit_potrf")


def posit_getrs(LU, ipiv, b, stream=None) -> None:
    """b <- A^{-1} b in place with the posit_getrf factors (one RHS, device tensors)."""
    import torch
    n, n2 = _mat(LU, "LU")
    if n2 < n:
        raise PositError(f"LU must be square, got {tuple(LU.shape)}")
    _vec(ipiv, "ipiv", torch.int32, n)
    _vec(b, "b", torch.int32, n)
    _check(lib().posit_getrs(b"N", n, _ptr(LU), _ld(LU), _ptr(ipiv), _ptr(b), _stream(stream)), "posit_getrs")


def posit_potrs(L, b, stream=None) -> None:
    """b <- A^{-1} b in place with the posit_potrf lower factor (one RHS, device tensors)."""
    import torch
    n, n2 = _mat(L, "L")
    if n2 < n:
        raise PositError(f"L must be square, got {tuple(L.shape)}")
    _vec(b, "b", torch.int32, n)
    _check(lib().posit_potrs(b"L", n, _ptr(L), _ld(L), _ptr(b), _stream(stream)), "posit_potrs")


def posit_iamax_key(col, global_row, row_min: int, key, stream=None) -> None:
    """key (int64 device tensor, 1) <- pivot key of the strided column view col (m x 1 or m) over rows
    whose global index (int32 device tensor, m) is >= row_min (see include/posit_b200.h)."""
    import torch
    if col.dtype != torch.int32 or not col.is_cuda:
        raise PositError("col: expected a CUDA torch.int32 column view")
    m = col.shape[0]
    stride = col.stride(0)
    _vec(global_row, "global_row", torch.int32, m)
    _vec(key, "key", torch.int64, 1)
    _check(lib().posit_iamax_key(m, _ptr(col), stride, _ptr(global_row), row_min, _ptr(key), _stream(stream)),
           "posit_iamax_key")


def posit_from_f64(x, out=None, stream=None):
    import torch
    _vec(x, "x", torch.float64, 0)
    if out is None:
        out = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    _vec(out, "out", torch.int32, x.numel())
    _check(lib().posit_from_f64(_ptr(x), _ptr(out), x.numel(), _stream(stream)), "posit_from_f64")
    return out


def posit_to_f64(p, out=None, stream=None):
    import torch
    _vec(p, "p", torch.int32, 0)
    if out is None:
        out = torch.empty(p.shape, dtype=torch.float64, device=p.device)
    _vec(out, "out", torch.float64, p.numel())
    _check(lib().posit_to_f64(_ptr(p), _ptr(out), p.numel(), _stream(stream)), "posit_to_f64")
    return out


def posit_vec_op(op: str, a, b=None, out=None, stream=None):
    import torch
    _vec(a, "a", torch.int32, 0)
    if b is not None:
        _vec(b, "b", torch.int32, a.numel())
    if out is None:
        out = torch.empty_like(a)
    _vec(out, "out", torch.int32, a.numel())
    _check(lib().posit_vec_op(OPS[op], _ptr(a), _ptr(a if b is None else b), _ptr(out), a.numel(), _stream(stream)),
           "posit_vec_op")
    return out


def posit_vec_dmac(c, a, b, out=None, stream=None):
    """out = c (+) (a (x) b) elementwise through the binary64-pipe MAC (posit_vec_dmac)."""
    import torch
    _vec(c, "c", torch.int32, 0)
    _vec(a, "a", torch.int32, c.numel())
    _vec(b, "b", torch.int32, c.numel())
    if out is None:
        out = torch.empty_like(c)
    _vec(out, "out", torch.int32, c.numel())
    _check(lib().posit_vec_dmac(_ptr(c), _ptr(a), _ptr(b), _ptr(out), c.numel(), _stream(stream)), "posit_vec_dmac")
    return out
