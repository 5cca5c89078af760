"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO posit arithmetic: it only draws binary64 matrices (and a
few raw bit-pattern sets) from numpy's PCG64 ``default_rng(seed)``.  Each side
converts binary64 -> posit32 with its own converter (oracle: ``or_from_f64``;
CUDA path: ``posit_from_f64``); the tests check that those conversions agree
bit for bit.

Recipes (BASELINE.json configs; reading Q14 -- row-major C-order
fill, successive draws from one generator):

  C1  rng(0).uniform(-1, 1, (256, 256))                         LU n=256 nb=32
  C2  rng(1): A, B, C = 3 x standard_normal((4096, 4096))         GEMM C -= A B
  C3  rng(2): G = standard_normal((8192, 8192)); A = G G^T / 8192 + I,
      lower copied to upper (symmetric to the bit)               Cholesky nb=256
  C4  rng(3).uniform(-1, 1, (16384, 16384))                      LU nb=256, 1..8 GPUs
  C5  rng(4).uniform(-1, 1, (8192, 8192)) scaled by 2^s, s in {-16,-4,0,4,16}

The paper's own workloads are N(0, sigma^2) random matrices (P:242, P:381,
P:483) and A = X^T X for Cholesky; there is no dataset.  Every
generator takes an optional size so parity tests can run the same recipe at
sizes the oracle finishes in seconds.
"""
from __future__ import annotations

import numpy as np

C1_N, C1_NB, C1_SEED = 256, 32, 0
C2_N, C2_SEED = 4096, 1
C3_N, C3_NB, C3_SEED = 8192, 256, 2
C4_N, C4_NB, C4_SEED = 16384, 256, 3
C5_N, C5_NB, C5_SEED = 8192, 256, 4
C5_SHIFTS = (-16, -4, 0, 4, 16)

# Operand ranges of Table tabrandom: [a, b)
RANGES = {
    "I0": (1.0, 2.0),
    "I1": (1e-38, 1e-30),
    "I2": (1e30, 1e38),
    "I3": (1e-15, 1e-14),
    "I4": (1e14, 1e15),
}


def lu_matrix(n: int = C1_N, seed: int = C1_SEED) -> np.ndarray:
    """U[-1,1) square matrix (configs 1, 4, 5 before scaling)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (n, n))


def config1(n: int = C1_N) -> np.ndarray:
    return lu_matrix(n, C1_SEED)


def config2(n: int = C2_N, m: int | None = None, k: int | None = None):
    """A (m x k), B (k x n), C (m x n), drawn in that order from rng(1)."""
    m = n if m is None else m
    k = n if k is None else k
    rng = np.random.default_rng(C2_SEED)
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((k, n))
    C = rng.standard_normal((m, n))
    return A, B, C


def config3(n: int = C3_N) -> np.ndarray:
    rng = np.random.default_rng(C3_SEED)
    G = rng.standard_normal((n, n))
    A = (G @ G.T) / n + np.eye(n)
    il = np.tril_indices(n, -1)
    A.T[il] = A[il]          # copy the lower triangle into the upper: symmetric to the bit
    return A


def config4(n: int = C4_N) -> np.ndarray:
    return lu_matrix(n, C4_SEED)


def config5(s: int, n: int = C5_N) -> np.ndarray:
    return np.ldexp(lu_matrix(n, C5_SEED), s)   # exact in binary64


def normal_matrix(shape, sigma: float = 1.0, seed: int = 0) -> np.ndarray:
    """N(0, sigma^2) as in the paper's GEMM and accuracy experiments."""
    return np.random.default_rng(seed).normal(0.0, sigma, shape)


def range_samples(label: str, count: int, seed: int = 0, signed: bool = True) -> np.ndarray:
    """Log-uniform draws from a Table-tabrandom range."""
    a, b = RANGES[label]
    rng = np.random.default_rng(seed)
    x = np.exp(rng.uniform(np.log(a), np.log(b), count))
    if signed:
        x *= np.where(rng.random(count) < 0.5, -1.0, 1.0)
    return x


def random_patterns(count: int, seed: int = 0) -> np.ndarray:
    """Uniformly random 32-bit patterns (covers every regime length, NaR, 0)."""
    return np.random.default_rng(seed).integers(0, 1 << 32, count, dtype=np.uint64).astype(np.uint32)


def edge_patterns() -> np.ndarray:
    """Structured posit32 bit patterns: every regime run length 1..31 with
    fraction-field fills {0, 1, LSB-only, all ones} and both signs, plus the
    reserved and extreme patterns.  Pure bit assembly (no rounding)."""
    out = {0x00000000, 0x80000000, 0x7FFFFFFF, 0x00000001, 0x40000000, 0x3FFFFFFF, 0x40000001}
    for run in range(1, 32):
        for ones in (0, 1):
            # magnitude bits after the sign: `run` copies of `ones`, then the opposite bit
            body_len = 31
            regime = ((1 << run) - 1) if ones else 0
            if run < body_len:
                regime = (regime << 1) | (0 if ones else 1)
                used = run + 1
            else:
                used = run
            rest = body_len - used
            fills = {0}
            if rest > 0:
                fills |= {1, (1 << rest) - 1, 1 << (rest - 1)}
            for f in fills:
                mag = (regime << rest) | f
                mag &= 0x7FFFFFFF
                if mag == 0:
                    continue
                out.add(mag)
                out.add((-mag) & 0xFFFFFFFF)
    return np.array(sorted(out), dtype=np.uint32)
