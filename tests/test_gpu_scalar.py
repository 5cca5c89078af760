"""GPU parity of the device scalar arithmetic (posit32.cuh) against the CPU
oracle, through the C ABI (posit_vec_op / posit_from_f64 / posit_to_f64).
Bit-exact on every word."""
import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import oracle as O
from tests.gpu_util import mismatch, to_dev, to_host

pytestmark = pytest.mark.gpu


def _operands(seed):
    parts = [SI.edge_patterns()]
    for i, lab in enumerate(SI.RANGES):
        parts.append(O.from_f64_array(SI.range_samples(lab, 20000, seed=seed + i)))
    parts.append(O.from_f64_array(SI.normal_matrix(50000, 1.0, seed=seed + 9)))
    parts.append(SI.random_patterns(100000, seed=seed + 10))
    return np.concatenate(parts)


@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "sqrt"])
def test_vec_ops_match_oracle(cuda_ok, op):
    import paper_2401_14117_b200 as PB
    ops = _operands(3)
    rng = np.random.default_rng(4)
    A = ops[rng.integers(0, ops.size, 400000)]
    B = ops[rng.integers(0, ops.size, 400000)]
    # near-cancellation pairs
    B[::3] = (-(A[::3].astype(np.int64) + rng.integers(-2, 3, A[::3].size))).astype(np.uint32)
    got = to_host(PB.posit_vec_op(op, to_dev(A), to_dev(B)))
    ref = O.vec_op(op, A, B)
    assert mismatch(got, ref) == 0


def test_exhaustive_posit8_lifted_pairs(cuda_ok):
    # all posit(8,0)-shaped extremes lifted to 32 bits: every pair of edge patterns
    import paper_2401_14117_b200 as PB
    E = SI.edge_patterns()
    A = np.repeat(E, E.size)
    B = np.tile(E, E.size)
    for op in ("add", "mul", "div"):
        assert mismatch(to_host(PB.posit_vec_op(op, to_dev(A), to_dev(B))), O.vec_op(op, A, B)) == 0


def test_from_to_f64_match_oracle(cuda_ok):
    import torch
    import paper_2401_14117_b200 as PB
    xs = np.concatenate([SI.normal_matrix(200000, 1.0, seed=1), SI.range_samples("I1", 20000), SI.range_samples("I2", 20000),
                         SI.range_samples("I3", 20000), SI.range_samples("I4", 20000), SI.lu_matrix(300, 2).ravel(),
                         np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e-300, 1e300, 2.0 ** 118, 2.0 ** -118,
                                   1.0 + 2.0 ** -28, 2.0 ** 113, 3 * 2.0 ** 114])])
    got = to_host(PB.posit_from_f64(torch.from_numpy(xs).cuda()))
    assert mismatch(got, O.from_f64_array(xs)) == 0
    got1 = to_host(PB.posit_from_f64(torch.from_numpy(xs).cuda()[1:]))    # 8-byte offset: the scalar path
    assert mismatch(got1, O.from_f64_array(xs[1:])) == 0
    pats = np.concatenate([SI.edge_patterns(), SI.random_patterns(300000, 5)])
    back = PB.posit_to_f64(to_dev(pats)).cpu().numpy()
    ref = O.to_f64_array(pats)
    assert np.array_equal(back, ref, equal_nan=True)
    back1 = PB.posit_to_f64(to_dev(pats)[1:]).cpu().numpy()
    assert np.array_equal(back1, ref[1:], equal_nan=True)


def test_exhaustive_roundtrip_2pow32_on_gpu(cuda_ok):
    # all 2^32 patterns: to_f64 -> from_f64 is the identity, on the device
    import torch
    import paper_2401_14117_b200 as PB
    chunk = 1 << 28
    bad = 0
    for c0 in range(0, 1 << 32, chunk):
        p = torch.arange(c0, c0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32)  # wraps to the bit pattern
        back = PB.posit_from_f64(PB.posit_to_f64(p))
        nar = p == torch.iinfo(torch.int32).min
        bad += int(((back != p) & ~nar).sum())
        del p, back
    assert bad == 0
