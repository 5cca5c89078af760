"""GPU parity of the binary64-pipe MAC (the D-MAC, csrc/gemm_d.cuh) against the
CPU oracle, one operation at a time, through the C ABI (posit_vec_op 'dadd' /
'dmul', posit_vec_dmac).  Bit-exact on every word.

The operand sets aim at the places where the D-MAC's argument could break
("the binary64-pipe MAC"):
* sums whose exact value needs more than 53 bits (exponent gaps 26..80), where
  binary64 RN would double-round: the round-to-odd pick must be right for both
  signs, including neighbours whose low word is all ones (a power of two minus
  a tiny value);
* exact lattice midpoints (ties to even) and near-midpoints at every gap 1..30;
* cancellation down to a few lattice steps, exact cancellation to zero;
* products whose RN(a*b) carries into the next binade (significands near
  sqrt(2) pairs) and products at every regime boundary of the scale range.
"""
import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import oracle as O
from tests.gpu_util import mismatch, to_dev, to_host

pytestmark = pytest.mark.gpu


def _pat(x):
    return O.from_f64_array(np.asarray(x, np.float64))


def _scaled(rng, n, emin, emax):
    """posits of random sign, fraction and binary scale in [emin, emax]."""
    e = rng.integers(emin, emax + 1, n)
    f = 1.0 + rng.random(n)
    s = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return _pat(s * f * np.exp2(e.astype(np.float64)))


def _sum_pairs(seed, n=200000):
    rng = np.random.default_rng(seed)
    parts_a, parts_b = [], []
    # far-apart exponents (inexact in binary64), both signs
    a = _scaled(rng, n, -40, 40)
    av = O.to_f64_array(a)
    gap = rng.integers(26, 81, n).astype(np.float64)
    b = _pat(np.where(rng.random(n) < 0.5, -1.0, 1.0) * np.abs(av) * (1.0 + rng.random(n)) * np.exp2(-gap))
    parts_a.append(a); parts_b.append(b)
    # powers of two (+-) against tiny values of either sign: neighbours with all-ones low words
    p2 = _pat(np.where(rng.random(n // 4) < 0.5, -1.0, 1.0) * np.exp2(rng.integers(-40, 41, n // 4).astype(np.float64)))
    tv = O.to_f64_array(p2)
    tiny = _pat(np.where(rng.random(n // 4) < 0.5, -1.0, 1.0) * np.abs(tv) * np.exp2(-rng.integers(26, 70, n // 4).astype(np.float64)) * (1.0 + rng.random(n // 4)))
    parts_a.append(p2); parts_b.append(tiny)
    # small gaps 0..30: ties and near-ties on the sum's lattice
    a = _scaled(rng, n, -40, 40)
    av = O.to_f64_array(a)
    gap = rng.integers(0, 31, n).astype(np.float64)
    b = _pat(np.where(rng.random(n) < 0.5, -1.0, 1.0) * np.abs(av) * (1.0 + rng.random(n)) * np.exp2(-gap))
    parts_a.append(a); parts_b.append(b)
    # cancellation: b = -a +- a few patterns, and exactly -a
    a = _scaled(rng, n // 2, -40, 40)
    d = rng.integers(-4, 5, n // 2)
    b = (-(a.astype(np.int64) + d)).astype(np.uint32)
    parts_a.append(a); parts_b.append(b)
    # the whole |E| <= 75 range (a product's range), random pairs
    parts_a.append(_scaled(rng, n, -75, 74)); parts_b.append(_scaled(rng, n, -75, 74))
    # outside the fast range (generic fallback): zeros, NaR, extremes
    E = SI.edge_patterns()
    parts_a.append(np.repeat(E, E.size)); parts_b.append(np.tile(E, E.size))
    return np.concatenate(parts_a), np.concatenate(parts_b)


def _mul_pairs(seed, n=300000):
    rng = np.random.default_rng(seed)
    parts_a, parts_b = [], []
    parts_a.append(_scaled(rng, n, -37, 36)); parts_b.append(_scaled(rng, n, -37, 36))
    # significand products near 2 (RN(a*b) may carry into the next binade)
    fa = 1.0 + rng.random(n) * 0.5 + 0.2
    fb = 2.0 / fa * (1.0 - rng.random(n) * 2.0 ** -rng.integers(20, 40, n))
    ea = rng.integers(-30, 30, n).astype(np.float64)
    eb = rng.integers(-6, 6, n).astype(np.float64)
    parts_a.append(_pat(fa * np.exp2(ea))); parts_b.append(_pat(-fb * np.exp2(eb)))
    # products at every regime boundary of the product scale (Ea + Eb = 4j - 1, 4j)
    j = rng.integers(-18, 19, n)
    ea = rng.integers(-37, 38, n)
    eb = np.clip(4 * j - ea - rng.integers(0, 2, n), -37, 36)
    parts_a.append(_pat((1.0 + rng.random(n)) * np.exp2(ea.astype(np.float64))))
    parts_b.append(_pat((1.0 + rng.random(n)) * np.exp2(eb.astype(np.float64))))
    # I0..I4 ranges and raw patterns (mostly outside the fast range: generic fallback)
    for i, lab in enumerate(SI.RANGES):
        parts_a.append(O.from_f64_array(SI.range_samples(lab, 20000, seed=seed + i)))
        parts_b.append(O.from_f64_array(SI.range_samples(lab, 20000, seed=seed + 7 + i)))
    parts_a.append(SI.random_patterns(50000, seed)); parts_b.append(SI.random_patterns(50000, seed + 1))
    return np.concatenate(parts_a), np.concatenate(parts_b)


def test_dadd_matches_oracle(cuda_ok):
    import paper_2401_14117_b200 as PB
    A, B = _sum_pairs(11)
    got = to_host(PB.posit_vec_op("dadd", to_dev(A), to_dev(B)))
    ref = O.vec_op("add", A, B)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(ref[i])) for i in bad[:8]]


def test_dmul_matches_oracle(cuda_ok):
    import paper_2401_14117_b200 as PB
    A, B = _mul_pairs(12)
    got = to_host(PB.posit_vec_op("dmul", to_dev(A), to_dev(B)))
    ref = O.vec_op("mul", A, B)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(ref[i])) for i in bad[:8]]


def test_dmac_matches_oracle(cuda_ok):
    """c (+) (a (x) b) with the accumulator anywhere in |E| <= 91 against the product."""
    import paper_2401_14117_b200 as PB
    rng = np.random.default_rng(13)
    A, B = _mul_pairs(14, n=200000)
    n = A.size
    P = O.vec_op("mul", A, B)
    pv = O.to_f64_array(P)
    kind = rng.integers(0, 5, n)
    gap = rng.integers(-60, 61, n).astype(np.float64)
    sgn = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    cv = np.where(kind == 0, -pv * (1.0 + (rng.random(n) - 0.5) * 2.0 ** -20),        # near cancellation
         np.where(kind == 1, sgn * np.abs(pv) * np.exp2(gap) * (1.0 + rng.random(n)),  # any gap
         np.where(kind == 2, sgn * np.exp2(rng.integers(-91, 92, n).astype(np.float64)) * (1.0 + rng.random(n)),
         np.where(kind == 3, -pv, rng.standard_normal(n) * 64.0))))
    cv = np.nan_to_num(cv, nan=1.0, posinf=1.0, neginf=-1.0)
    C = _pat(cv)
    got = to_host(PB.posit_vec_dmac(to_dev(C), to_dev(A), to_dev(B)))
    ref = O.vec_op("add", C, P)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(hex(C[i]), hex(A[i]), hex(B[i]), hex(got[i]), hex(ref[i])) for i in bad[:8]]


def _div_pairs(seed, n=300000):
    """dividends over the accumulator range, divisors over the operand range, plus
    quotients built to sit on or next to a lattice midpoint / lattice point."""
    rng = np.random.default_rng(seed)
    parts_a, parts_b = [], []
    parts_a.append(_scaled(rng, n, -75, 74)); parts_b.append(_scaled(rng, n, -37, 36))
    # a = q (x) b exactly or a few patterns off: the quotient is a lattice point / near one
    q = _scaled(rng, n, -30, 30)
    b = _scaled(rng, n, -30, 30)
    a = O.vec_op("mul", q, b)
    d = rng.integers(-3, 4, n)
    parts_a.append((a.astype(np.int64) + d).astype(np.uint32)); parts_b.append(b)
    # quotients next to a midpoint of the quotient's lattice: a = (q + half a step) * b rounded
    qv = O.to_f64_array(q)
    qn = O.to_f64_array((q.astype(np.int64) + 1).astype(np.uint32))
    mid = 0.5 * (qv + qn) * (1.0 + (rng.random(n) - 0.5) * np.exp2(-rng.integers(24, 50, n).astype(np.float64)))
    parts_a.append(_pat(mid * O.to_f64_array(b))); parts_b.append(b)
    # small-integer and power-of-two divisors (exact quotients, long carries)
    parts_a.append(_scaled(rng, n // 2, -60, 60))
    parts_b.append(_pat(np.where(rng.random(n // 2) < 0.5, -1.0, 1.0) * rng.integers(1, 64, n // 2).astype(np.float64)
                        * np.exp2(rng.integers(-20, 21, n // 2).astype(np.float64))))
    # Cholesky-like: |a| <~ |b|, b > 0 near 1 (l_ik = a_ik / l_kk)
    parts_a.append(_pat(rng.standard_normal(n) * 0.05)); parts_b.append(_pat(1.0 + 0.2 * rng.random(n)))
    # outside the fast range (generic fallback): zeros, NaR, extremes, raw patterns
    E = SI.edge_patterns()
    parts_a.append(np.repeat(E, E.size)); parts_b.append(np.tile(E, E.size))
    parts_a.append(SI.random_patterns(50000, seed)); parts_b.append(SI.random_patterns(50000, seed + 1))
    return np.concatenate(parts_a), np.concatenate(parts_b)


def test_ddiv_matches_oracle(cuda_ok):
    """The panel kernels' binary64-pipe division (pld::div_r), one operation at a time."""
    import paper_2401_14117_b200 as PB
    A, B = _div_pairs(15)
    got = to_host(PB.posit_vec_op("ddiv", to_dev(A), to_dev(B)))
    ref = O.vec_op("div", A, B)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(ref[i])) for i in bad[:8]]


def test_dsqrt_matches_oracle(cuda_ok):
    """The cluster potf2's binary64-pipe square root (pld::sqrt_r): random arguments over
    |E| <= 75, exact squares and their pattern neighbours, arguments whose root sits
    next to a midpoint of the root's lattice, and the generic fallback."""
    import paper_2401_14117_b200 as PB
    rng = np.random.default_rng(16)
    n = 400000
    parts = [_scaled(rng, n, -75, 74)]
    r = _scaled(rng, n, -37, 36)
    sq = O.vec_op("mul", r, r)                                   # rounded squares
    parts.append((sq.astype(np.int64) + rng.integers(-3, 4, n)).astype(np.uint32))
    r14 = _pat(rng.integers(1, 1 << 13, n).astype(np.float64) * np.exp2(rng.integers(-30, 20, n).astype(np.float64)))
    parts.append(O.vec_op("mul", r14, r14))                      # exact squares (13-bit roots)
    rv = np.abs(O.to_f64_array(r))
    rn = np.abs(O.to_f64_array((r.astype(np.int64) + 1).astype(np.uint32)))
    mid = 0.5 * (rv + rn) * (1.0 + (rng.random(n) - 0.5) * np.exp2(-rng.integers(24, 50, n).astype(np.float64)))
    parts.append(_pat(mid * mid))
    parts.append(_pat(1.0 + rng.random(n) * 3.0))                # Cholesky diagonals of configs[2]
    parts.append(SI.edge_patterns()); parts.append(SI.random_patterns(100000, 17))
    A = np.concatenate(parts)
    got = to_host(PB.posit_vec_op("dsqrt", to_dev(A)))
    ref = O.vec_op("sqrt", A, A)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, [(hex(A[i]), hex(got[i]), hex(ref[i])) for i in bad[:8]]


@pytest.mark.parametrize("path", ["0", "1"])
def test_gemm_paths_identical_bits(cuda_ok, tmp_path, path):
    """The integer-MAC and binary64-MAC kernels give the oracle's bits on a GEMM
    with extreme operands mixed in (slabs that take the generic path)."""
    import os
    import subprocess
    import sys
    rng = np.random.default_rng(15)
    m, n, k = 200, 264, 150
    A = _pat(rng.standard_normal((m, k)) * np.exp2(rng.integers(-12, 13, (m, k))))
    B = _pat(rng.standard_normal((k, n)) * np.exp2(rng.integers(-12, 13, (k, n))))
    C = _pat(rng.standard_normal((m, n)) * 100.0)
    A[5, 17] = 0
    B[80, 3] = 0x7FFFFF00                          # |E| > 37: that slab runs the generic path
    ref = O.gemm(A, B, C)
    src = tmp_path / "in.npz"
    np.savez(src, A=A, B=B, C=C)
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_2401_14117_b200 as PB; "
            "from tests.gpu_util import to_dev, to_host; d = np.load(%r); C = to_dev(d['C']); "
            "PB.posit_gemm(to_dev(d['A']), to_dev(d['B']), C); np.save(%r, to_host(C))") % (
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), str(src), str(tmp_path / "out.npy"))
    env = dict(os.environ, POSIT_GEMM_PATH=path)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert mismatch(np.load(tmp_path / "out.npy"), ref) == 0
