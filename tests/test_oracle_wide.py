"""S:443's counts: the C oracle's posit32 add / sub / mul / div on >= 1e7
random pairs each and sqrt on >= 1e6 samples, against the exact checker.

The checker here is oracle/checker_wide.c: checker.py's definitions (Eq.1
value P:123-138, bisection over the signed pattern order S:37, the (n+1)-bit
midpoint rule of SURVEY 8(c) c2, readings Q1-Q3) with exact 768-bit integer
comparisons instead of Fractions.  It is first pinned to checker.py itself
(exhaustive posit(8, es) and random posit32), then used on the big samples.

Operand mix (all seeded): uniformly random 32-bit patterns (every regime
length, NaR, 0), N(0,1) and Table tabrandom ranges I0..I4,
nearby-magnitude pairs of opposite sign (cancellation), and far-apart pairs
whose exponents of their last fraction bits differ by more than 90 (the
oracle's "entirely below the guard position" branch, posit_oracle.c or_add).
"""
import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import checker as X
from oracle import checker_wide as W
from oracle import oracle as O


def test_checker_wide_equals_fraction_checker_posit8_exhaustive():
    pats = np.arange(256, dtype=np.uint32)
    A, B = (m.ravel() for m in np.meshgrid(pats, pats))
    for es in (0, 1, 2):
        for op in ("add", "sub", "mul", "div"):
            want, _ = W.expected(op, A, B, n=8, es=es)
            f = getattr(X, op)
            assert all(f(a, b, 8, es) == w for a, b, w in zip(A.tolist(), B.tolist(), want.tolist())), (op, es)
        want, _ = W.expected("sqrt", pats, n=8, es=es)
        assert all(X.sqrt(a, 8, es) == w for a, w in zip(pats.tolist(), want.tolist()))


def test_checker_wide_equals_fraction_checker_posit32():
    ops = np.concatenate([SI.edge_patterns(), SI.random_patterns(1500, seed=41),
                          O.from_f64_array(SI.normal_matrix(500, 1.0, seed=42))])
    rng = np.random.default_rng(43)
    A = ops[rng.integers(0, ops.size, 1500)]
    B = ops[rng.integers(0, ops.size, 1500)]
    for op in ("add", "sub", "mul", "div"):
        want, _ = W.expected(op, A, B)
        f = getattr(X, op)
        assert all(f(a, b) == w for a, b, w in zip(A.tolist(), B.tolist(), want.tolist())), op
    want, _ = W.expected("sqrt", ops)
    assert all(X.sqrt(a) == w for a, w in zip(ops.tolist(), want.tolist()))


def _mix(count: int, seed: int):
    """count operand pairs: 40% raw patterns, 20% N(0,1), 20% I0..I4, 10% near-equal
    opposite-sign, 10% far apart (|X_x - X_y| > 90)."""
    rng = np.random.default_rng(seed)
    q = count // 10
    A = [SI.random_patterns(4 * q, seed=seed + 1)]
    B = [SI.random_patterns(4 * q, seed=seed + 2)]
    A.append(O.from_f64_array(SI.normal_matrix(2 * q, 1.0, seed=seed + 3)))
    B.append(O.from_f64_array(SI.normal_matrix(2 * q, 1.0, seed=seed + 4)))
    labs = list(SI.RANGES)
    for i in range(2):
        parts = [O.from_f64_array(SI.range_samples(labs[(j + i) % 5], 2 * q // 5 + 1, seed=seed + 10 + 5 * i + j))
                 for j in range(5)]
        (A if i == 0 else B).append(np.concatenate(parts)[: 2 * q])
    a = SI.random_patterns(q, seed=seed + 5)
    d = rng.integers(-4, 5, q)
    A.append(a)
    B.append((-(a.astype(np.int64) + d)).astype(np.uint32))          # -(a + small): cancellation
    big = np.ldexp(rng.uniform(1.0, 2.0, q), rng.integers(40, 119, q)) * rng.choice([-1.0, 1.0], q)
    small = np.ldexp(rng.uniform(1.0, 2.0, q), rng.integers(-119, -40, q)) * rng.choice([-1.0, 1.0], q)
    swap = rng.random(q) < 0.5
    A.append(O.from_f64_array(np.where(swap, small, big)))
    B.append(O.from_f64_array(np.where(swap, big, small)))
    A, B = np.concatenate(A), np.concatenate(B)
    perm = rng.permutation(A.size)
    return A[perm], B[perm]


@pytest.mark.slow
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div"])
def test_oracle_1e7_pairs_vs_exact_checker(op):
    # ">= 1e7 random pairs" per operation against the exact rational definition
    A, B = _mix(10_000_000, seed={"add": 100, "sub": 200, "mul": 300, "div": 400}[op])
    assert A.size >= 10_000_000
    got = O.vec_op(op, A, B)
    want, nbad = W.expected(op, A, B, got)
    bad = np.nonzero(want != got)[0][:5]
    assert nbad == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(want[i])) for i in bad]


@pytest.mark.slow
def test_oracle_sqrt_1e6_vs_exact_checker():
    # ">= 1e6" sqrt samples (every regime: raw patterns; plus N(0,1)^2-like and I0..I4 values)
    parts = [SI.random_patterns(2_000_000, seed=501), O.from_f64_array(np.abs(SI.normal_matrix(500_000, 1.0, seed=502)))]
    parts += [O.from_f64_array(SI.range_samples(lab, 100_000, seed=503 + i, signed=False))
              for i, lab in enumerate(SI.RANGES)]
    A = np.concatenate(parts)
    got = O.vec_op("sqrt", A)
    want, nbad = W.expected("sqrt", A, None, got)
    bad = np.nonzero(want != got)[0][:5]
    assert nbad == 0, [(hex(A[i]), hex(got[i]), hex(want[i])) for i in bad]


def test_far_apart_pairs_reach_the_oracle_shortcut():
    # the far-apart share of _mix really has |X_x - X_y| > 90 (X = scale - f_s, the
    # exponent of the last fraction bit): count them with the oracle's own decode helpers
    A, B = _mix(20_000, seed=7)
    Xa = np.array([O.scale(int(a)) - O.fraction_bits(int(a)) for a in A[:20_000]])
    Xb = np.array([O.scale(int(b)) - O.fraction_bits(int(b)) for b in B[:20_000]])
    ok = (A != 0) & (B != 0) & (A != 0x80000000) & (B != 0x80000000)
    far = int(np.count_nonzero(ok & (np.abs(Xa - Xb) > 90)))
    assert far >= 1500, far
