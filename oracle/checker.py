"""Exact-rational checker for posit(n, es) arithmetic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of both the C
oracle and the CUDA path: it shares no code with either.

It states the definitions in their most literal form:

* ``value(p)``   -- Eq.1 of the paper: sign, regime run k(r),
  es exponent bits (missing bits read as 0), remaining bits the fraction
  (the exact fraction budget, reading Q5 / S:39-45), as a ``Fraction``.
* ``round_to_posit(x)`` -- round-to-nearest-even on the encoding (reading Q1,
  S:70) stated without any bit manipulation: find by bisection over the
  signed order of patterns the largest pattern p with value(p) <= |x|;
  the midpoint between p and p+1 is the value of the pattern 2p+1 read as a
  Posit(n+1, es); below it -> p, above -> p+1, equal -> the
  even one of p, p+1.  |x| >= maxpos -> maxpos, 0 < |x| <= minpos -> minpos
  (reading Q2).
* add/sub/mul/div: exact rational result, rounded once.
* sqrt: the largest p with value(p)^2 <= x, then the midpoint compared by
  squares -- all rational.
"""
from __future__ import annotations

import functools
from fractions import Fraction

NAR = None  # value() returns None for NaR


@functools.lru_cache(maxsize=1 << 20)
def value(p: int, n: int = 32, es: int = 2):
    mask = (1 << n) - 1
    p &= mask
    if p == 0:
        return Fraction(0)
    if p == 1 << (n - 1):
        return NAR
    sign = p >> (n - 1)
    if sign:
        p = (-p) & mask
    bits = [(p >> i) & 1 for i in range(n - 2, -1, -1)]  # after the sign, MSB first
    r = bits[0]
    m = 0
    while m < len(bits) and bits[m] == r:
        m += 1
    k = m - 1 if r == 1 else -m
    rest = bits[m + 1:]  # skip the terminating bit (if any)
    e = 0
    for j in range(es):
        e = 2 * e + (rest[j] if j < len(rest) else 0)
    frac_bits = rest[es:]
    f = Fraction(0)
    for j, b in enumerate(frac_bits):
        if b:
            f += Fraction(1, 2 ** (j + 1))
    useed = 2 ** (2 ** es)
    v = Fraction(useed) ** k * Fraction(2) ** e * (1 + f)
    return -v if sign else v


def maxpos(n: int = 32) -> int:
    return (1 << (n - 1)) - 1


def _largest_le(ax: Fraction, n: int, es: int) -> int:
    lo, hi = 1, maxpos(n)  # value(lo) <= ax < value(hi) maintained by the callers' range checks
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if value(mid, n, es) <= ax:
            lo = mid
        else:
            hi = mid
    return lo


def round_to_posit(x: Fraction, n: int = 32, es: int = 2) -> int:
    mask = (1 << n) - 1
    if x == 0:
        return 0
    ax = abs(x)
    mp = maxpos(n)
    if ax >= value(mp, n, es):
        p = mp
    elif ax <= value(1, n, es):
        p = 1
    else:
        p = _largest_le(ax, n, es)
        if value(p, n, es) != ax:
            mid = value(2 * p + 1, n + 1, es)
            if ax > mid or (ax == mid and (p & 1)):
                p = p + 1
    return ((-p) & mask) if x < 0 else p


def _nar(n):
    return 1 << (n - 1)


def add(a: int, b: int, n: int = 32, es: int = 2) -> int:
    va, vb = value(a, n, es), value(b, n, es)
    if va is NAR or vb is NAR:
        return _nar(n)
    return round_to_posit(va + vb, n, es)


def sub(a: int, b: int, n: int = 32, es: int = 2) -> int:
    va, vb = value(a, n, es), value(b, n, es)
    if va is NAR or vb is NAR:
        return _nar(n)
    return round_to_posit(va - vb, n, es)


def mul(a: int, b: int, n: int = 32, es: int = 2) -> int:
    va, vb = value(a, n, es), value(b, n, es)
    if va is NAR or vb is NAR:
        return _nar(n)
    return round_to_posit(va * vb, n, es)


def div(a: int, b: int, n: int = 32, es: int = 2) -> int:
    va, vb = value(a, n, es), value(b, n, es)
    if va is NAR or vb is NAR or vb == 0:
        return _nar(n)
    return round_to_posit(va / vb, n, es)


def sqrt(a: int, n: int = 32, es: int = 2) -> int:
    va = value(a, n, es)
    if va is NAR or va < 0:
        return _nar(n)
    if va == 0:
        return 0
    mp = maxpos(n)
    if va >= value(mp, n, es) ** 2:
        return mp
    if va <= value(1, n, es) ** 2:
        return 1
    lo, hi = 1, mp
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if value(mid, n, es) ** 2 <= va:
            lo = mid
        else:
            hi = mid
    p = lo
    if value(p, n, es) ** 2 == va:
        return p
    m = value(2 * p + 1, n + 1, es)
    if va > m * m or (va == m * m and (p & 1)):
        p += 1
    return p


def from_float(x: float, n: int = 32, es: int = 2) -> int:
    if x != x or x in (float("inf"), float("-inf")):
        return _nar(n)
    return round_to_posit(Fraction(x), n, es)
