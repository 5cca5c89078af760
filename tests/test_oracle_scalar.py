"""Pins of the C oracle's scalar Posit arithmetic against what the paper, the
spec's worked examples and exact rational arithmetic fix.

Citations: P:n = PAPER.md line n; S:n = SPEC.md line n.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import checker as X
from oracle import oracle as O

ONE, TWO, MONE, NAR, MAXPOS, MINPOS = 0x40000000, 0x48000000, 0xC0000000, 0x80000000, 0x7FFFFFFF, 0x00000001


def test_format_constants():
    # Eq.1: u = 2^(2^es) = 16 for Posit(32,2)
    assert O.from_f64(1.0) == ONE
    assert O.from_f64(2.0) == TWO
    assert O.from_f64(4.0) == 0x50000000
    assert O.from_f64(16.0) == 0x60000000         # useed: regime "110"
    assert O.from_f64(-1.0) == MONE
    assert O.from_f64(0.5) == 0x38000000
    assert O.from_f64(2.0 ** -27) == 0x00A00000   # k = -7, e = 1
    assert O.to_f64(MAXPOS) == 2.0 ** 120         # 16^30
    assert O.to_f64(MINPOS) == 2.0 ** -120
    assert math.isnan(O.to_f64(NAR))
    assert O.from_f64(float("nan")) == NAR and O.from_f64(float("inf")) == NAR
    assert O.from_f64(-0.0) == 0


def test_checker_value_definition():
    # the checker's Eq.1 at hand-derived points (posit(8,0): useed 2)
    assert X.value(0x40, 8, 0) == 1 and X.value(0x7F, 8, 0) == 64 and X.value(0x01, 8, 0) == Fraction(1, 64)
    assert X.value(0x60, 8, 0) == 2 and X.value(0x50, 8, 0) == Fraction(3, 2)
    assert X.value(ONE) == 1 and X.value(MAXPOS) == 2 ** 120 and X.value(MINPOS) == Fraction(1, 2 ** 120)
    assert X.value(NAR) is None and X.value(0) == 0
    # truncated exponent zone: 0x7FFFFFFD has k=28, e bits '1'+missing -> 2^114
    assert X.value(0x7FFFFFFD) == 2 ** 114 and X.value(0x7FFFFFFE) == 2 ** 116


def test_fraction_bits_match_paper():
    # f_s = 27 on I0 = [1,2), eps = 2^-27 ~ 7.5e-9
    for x in SI.range_samples("I0", 200, seed=1, signed=False):
        assert O.fraction_bits(O.from_f64(x)) == 27
    assert O.to_f64(ONE + 1) - 1.0 == 2.0 ** -27
    # on I1 and I2 f_s ranges from 0 to 3 (beyond maxpos/minpos -> saturated, f_s = 0)
    for lab in ("I1", "I2"):
        fs = {O.fraction_bits(O.from_f64(x)) for x in SI.range_samples(lab, 2000, seed=2, signed=False)}
        assert fs <= {0, 1, 2, 3} and 3 in fs and 0 in fs
    # derived: f_s in {15, 16} on I3 and I4
    for lab in ("I3", "I4"):
        fs = {O.fraction_bits(O.from_f64(x)) for x in SI.range_samples(lab, 2000, seed=3, signed=False)}
        assert fs <= {15, 16}


def test_spec_worked_examples():
    assert O.add(ONE, ONE) == TWO
    assert O.from_f64(1.0 + 2.0 ** -28) == ONE                      # S:75 tie -> even
    assert O.from_f64(1.0 + 3 * 2.0 ** -28) == ONE + 2              # tie -> even (up)
    assert O.from_f64(2.0 ** 122) == MAXPOS
    p61 = O.from_f64(2.0 ** 61)
    assert O.mul(p61, p61) == MAXPOS
    assert O.div(ONE, 0) == NAR
    assert O.sqrt(O.from_f64(4.0)) == TWO
    assert O.sqrt(MONE) == NAR
    assert O.neg(ONE) == MONE and O.neg(NAR) == NAR and O.neg(0) == 0
    assert O.from_f64(2.0 ** -130) == MINPOS and O.from_f64(-(2.0 ** -130)) == (-MINPOS) & 0xFFFFFFFF
    for p in SI.edge_patterns().tolist():
        if p == NAR:
            continue
        assert O.add(p, 0) == p and O.mul(p, ONE) == p and O.div(p, ONE) == p
    assert O.div(ONE, O.from_f64(3.0)) == X.div(ONE, O.from_f64(3.0))
    assert O.sqrt(TWO) == X.sqrt(TWO)


def test_truncated_zone_rounding_reading_Q1():
    # RNE on the encoding: between 2^116 (0x7FFFFFFE) and maxpos the midpoint is 2^118
    assert O.from_f64(1.01 * 2.0 ** 118) == MAXPOS
    assert O.from_f64(2.0 ** 118) == 0x7FFFFFFE        # tie -> even pattern
    assert O.from_f64(1.9 * 2.0 ** 117) == 0x7FFFFFFE
    assert O.from_f64(2.0 ** -118) == 0x00000002        # mirror: midpoint of minpos and 2^-116 -> even
    for x in (2.0 ** 113, 1.5 * 2.0 ** 113, 2.0 ** 115, 3 * 2.0 ** 114, 2.0 ** -113, 2.0 ** -115, 1.3 * 2.0 ** -119):
        assert O.from_f64(x) == X.from_float(x)
        assert O.from_f64(-x) == X.from_float(-x)


@pytest.mark.parametrize("es", [0, 1, 2])
def test_exhaustive_posit8_vs_exact_rationals(es):
    # S:144 / S:443: exhaustive at width 8 against the exact-rational checker
    bad = []
    pats = np.arange(256, dtype=np.uint32)
    A = np.repeat(pats, 256)
    B = np.tile(pats, 256)
    for op in ("add", "sub", "mul", "div"):
        got = O.vec_op(op, A, B, n=8, es=es)
        f = getattr(X, op)
        for a, b, g in zip(A.tolist(), B.tolist(), got.tolist()):
            if f(a, b, 8, es) != g:
                bad.append((op, a, b, g))
    got = O.vec_op("sqrt", pats, n=8, es=es)
    for a, g in zip(pats.tolist(), got.tolist()):
        if X.sqrt(a, 8, es) != g:
            bad.append(("sqrt", a, g))
    assert not bad, bad[:10]


def _posit32_operands(seed: int) -> np.ndarray:
    parts = [SI.edge_patterns()]
    for i, lab in enumerate(SI.RANGES):
        parts.append(O.from_f64_array(SI.range_samples(lab, 300, seed=seed + i)))
    parts.append(O.from_f64_array(SI.normal_matrix(600, 1.0, seed=seed + 9)))
    parts.append(SI.random_patterns(600, seed=seed + 10))
    return np.concatenate(parts)


def test_random_posit32_vs_exact_rationals():
    # correct rounding vs the exact-rational oracle; structured + I0..I4 + raw
    ops = _posit32_operands(100)
    rng = np.random.default_rng(7)
    A = ops[rng.integers(0, ops.size, 2500)]
    B = ops[rng.integers(0, ops.size, 2500)]
    # nearby-magnitude pairs exercise cancellation
    B2 = (A.astype(np.int64) + rng.integers(-3, 4, A.size)).astype(np.uint32)
    B2 = np.where(rng.random(A.size) < 0.5, B2, (-B2.astype(np.int64)).astype(np.uint32))
    bad = []
    for op in ("add", "sub", "mul", "div"):
        for BB in (B, B2):
            got = O.vec_op(op, A, BB)
            f = getattr(X, op)
            for a, b, g in zip(A.tolist(), BB.tolist(), got.tolist()):
                if f(a, b) != g:
                    bad.append((op, hex(a), hex(b), hex(g)))
    got = O.vec_op("sqrt", ops)
    for a, g in zip(ops.tolist(), got.tolist()):
        if X.sqrt(a) != g:
            bad.append(("sqrt", hex(a), hex(g)))
    assert not bad, bad[:10]


def test_from_f64_vs_exact_rationals():
    xs = np.concatenate([SI.normal_matrix(500, 1.0, seed=3), SI.range_samples("I1", 200), SI.range_samples("I2", 200),
                         SI.range_samples("I3", 200), SI.range_samples("I4", 200),
                         np.array([2.0 ** 118, 2.0 ** 113, 1e-300, 1e300, 5e-324, 1.0 + 2 ** -28])])
    got = O.from_f64_array(xs)
    for x, g in zip(xs.tolist(), got.tolist()):
        assert X.from_float(x) == g, (x, hex(g))


def test_negation_symmetry_and_order():
    # op(-p, -q) = -op(p, q); value order = signed pattern order
    ops = _posit32_operands(5)
    rng = np.random.default_rng(11)
    A = ops[rng.integers(0, ops.size, 4000)]
    B = ops[rng.integers(0, ops.size, 4000)]
    nA, nB = O.vec_op("neg", A), O.vec_op("neg", B)
    assert np.array_equal(O.vec_op("add", nA, nB), O.vec_op("neg", O.vec_op("add", A, B)))
    assert np.array_equal(O.vec_op("mul", nA, B), O.vec_op("neg", O.vec_op("mul", A, B)))
    assert np.array_equal(O.vec_op("mul", nA, nB), O.vec_op("mul", A, B))
    assert np.array_equal(O.vec_op("div", nA, B), O.vec_op("neg", O.vec_op("div", A, B)))
    s = np.unique(ops.view(np.int32))
    s = s[s != np.int32(-(2 ** 31))]
    v = O.to_f64_array(s.view(np.uint32))
    assert np.all(np.diff(v) > 0)


@pytest.mark.slow
def test_exhaustive_roundtrip_all_2pow32():
    # BASELINE north_star / S:141 / S:442: all 2^32 patterns through to_f64 -> from_f64,
    # and adjacent patterns strictly increasing in value
    bad, unordered = O.roundtrip_all32()
    assert bad == 0 and unordered == 0
