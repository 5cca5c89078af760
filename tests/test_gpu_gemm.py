"""GPU parity of posit_gemm / posit_syrk (the hot path) with the CPU oracle,
element by element, through the C ABI.  Sizes span several 64x128 tiles and
16-deep k-slabs with ragged tails; the full config-2 size is checked on
sampled outputs the oracle computes one by one."""
import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import oracle as O
from tests.gpu_util import mismatch, to_dev, to_host

pytestmark = pytest.mark.gpu

ONE, MONE = O.P32_ONE, O.P32_MONE


def _pats(x):
    return O.from_f64_array(x)


def _gpu_gemm(A, B, C, transb="N", alpha=MONE, beta=ONE, naive=False, transa="N"):
    import paper_2401_14117_b200 as PB
    dA, dB, dC = to_dev(A), to_dev(B), to_dev(C)
    f = PB.posit_gemm_naive if naive else PB.posit_gemm
    f(dA, dB, dC, transb=transb, alpha=alpha, beta=beta, transa=transa)
    return to_host(dC)


SHAPES = [(1, 1, 1), (3, 5, 7), (64, 128, 16), (67, 131, 45), (130, 257, 64), (200, 129, 300), (257, 300, 33)]


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("transb", ["N", "T"])
def test_gemm_matches_oracle(cuda_ok, m, n, k, transb):
    A, B, C = SI.config2(n=n, m=m, k=k)
    if transb == "T":
        B = B.T.copy()
    A, B, C = _pats(A), _pats(B), _pats(C)
    ref = O.gemm(A, B, C, transb=transb)
    assert mismatch(_gpu_gemm(A, B, C, transb), ref) == 0
    assert mismatch(_gpu_gemm(A, B, C, transb, naive=True), ref) == 0


@pytest.mark.parametrize("m,n,k", [(3, 5, 7), (67, 131, 45), (200, 129, 300)])
@pytest.mark.parametrize("transa", ["N", "T"])
@pytest.mark.parametrize("transb", ["N", "T"])
def test_gemm_four_transpose_variants(cuda_ok, m, n, k, transa, transb):
    # Eq.2 with op(X) in {X, X^T}: A stored m x k or k x m, B k x n or n x k
    A, B, C = SI.config2(n=n, m=m, k=k)
    if transa == "T":
        A = A.T.copy()
    if transb == "T":
        B = B.T.copy()
    A, B, C = _pats(A), _pats(B), _pats(C)
    ref = O.gemm(A, B, C, transa=transa, transb=transb)
    assert mismatch(_gpu_gemm(A, B, C, transb, transa=transa), ref) == 0
    assert mismatch(_gpu_gemm(A, B, C, transb, transa=transa, naive=True), ref) == 0


@pytest.mark.parametrize("alpha,beta", [(ONE, ONE), (ONE, 0), (MONE, 0)])
def test_gemm_alpha_beta(cuda_ok, alpha, beta):
    A, B, C = SI.config2(n=96, m=70, k=50)
    A, B, C = _pats(A), _pats(B), _pats(C)
    assert mismatch(_gpu_gemm(A, B, C, alpha=alpha, beta=beta), O.gemm(A, B, C, alpha=alpha, beta=beta)) == 0


@pytest.mark.parametrize("m,n,k", [(70, 140, 80), (300, 520, 80)])
def test_gemm_special_values_and_cancellation(cuda_ok, m, n, k):
    # zeros, NaR, huge/tiny magnitudes (slow k-slabs), exact cancellations (integers);
    # 300 x 520 is above the one-thread-per-output cutoff, so the tiled k_gemm's
    # generic slab and thread-recompute paths run (70 x 140 takes k_gemm_tiny)
    rng = np.random.default_rng(3)
    A = rng.integers(-3, 4, (m, k)).astype(np.float64)
    B = rng.integers(-3, 4, (k, n)).astype(np.float64)
    C = rng.integers(-5, 6, (m, n)).astype(np.float64)
    A, B, C = _pats(A), _pats(B), _pats(C)
    assert mismatch(_gpu_gemm(A, B, C), O.gemm(A, B, C)) == 0
    A2 = _pats(SI.normal_matrix((m, k), 1.0, 4))
    A2[5, 7] = O.P32_NAR
    A2[9, :] = 0
    A2[11, 3] = O.from_f64(1e30)
    A2[12, 40] = O.from_f64(1e-33)
    B2 = _pats(SI.normal_matrix((k, n), 1e3, 5))
    C2 = _pats(SI.normal_matrix((m, n), 1e20, 6))        # accumulators beyond the fast range
    C2[:, 0] = O.from_f64(2.0 ** 110)
    assert mismatch(_gpu_gemm(A2, B2, C2), O.gemm(A2, B2, C2)) == 0


@pytest.mark.parametrize("sigma", [1e-2, 1.0, 1e2, 1e4, 1e6])
def test_gemm_sigma_sweep(cuda_ok, sigma):
    # Fig gemm_v100's operand scales: same bits at every sigma
    A = _pats(SI.normal_matrix((90, 60), sigma, 1))
    B = _pats(SI.normal_matrix((60, 150), sigma, 2))
    C = _pats(SI.normal_matrix((90, 150), sigma, 3))
    assert mismatch(_gpu_gemm(A, B, C), O.gemm(A, B, C)) == 0


def test_gemm_config2_full_size_sampled(cuda_ok):
    # configs[1]: m=n=k=4096, N(0,1) seed 1, C -= A B; the oracle computes 24 x 24 sampled outputs
    import torch
    import paper_2401_14117_b200 as PB
    A, B, C = SI.config2()
    dA = PB.posit_from_f64(torch.from_numpy(A).cuda())
    dB = PB.posit_from_f64(torch.from_numpy(B).cuda())
    dC = PB.posit_from_f64(torch.from_numpy(C).cuda())
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(4096, 24, replace=False))
    cols = np.sort(rng.choice(4096, 24, replace=False))
    # the conversion itself must agree with the oracle's on the sampled operands
    Ap, Bp, Cp = _pats(A[rows]), _pats(B[:, cols]), _pats(C[np.ix_(rows, cols)])
    assert mismatch(to_host(dA)[rows], Ap) == 0
    PB.posit_gemm(dA, dB, dC)
    got = to_host(dC)[np.ix_(rows, cols)]
    assert mismatch(got, O.gemm(Ap, Bp, Cp)) == 0


def test_syrk_matches_oracle_and_keeps_upper(cuda_ok):
    import paper_2401_14117_b200 as PB
    for n, k in [(1, 3), (70, 33), (200, 256), (129, 17)]:
        A = _pats(SI.normal_matrix((n, k), 1.0, n))
        C = _pats(SI.config3(n))
        ref = O.syrk_lower(A, C)
        dC = to_dev(C)
        PB.posit_syrk(to_dev(A), dC)
        got = to_host(dC)
        assert mismatch(got, ref) == 0


def test_gemm_bad_arguments(cuda_ok):
    import paper_2401_14117_b200 as PB
    A = to_dev(_pats(np.ones((4, 4))))
    with pytest.raises(PB.PositError):
        PB.posit_gemm(A, A, A, alpha=O.from_f64(2.0))
    with pytest.raises(PB.PositError):
        PB.posit_gemm(A, A, A, beta=O.from_f64(0.5))


@pytest.mark.parametrize("m,n", [(70, 130), (300, 520)])
@pytest.mark.parametrize("ea,ec", [(36, 88), (38, 92), (-36, -100), (-38, 40), (30, 100)])
def test_gemm_fast_path_range_boundaries(cuda_ok, ea, ec, m, n):
    # operand scales straddling the staging limit (|E| <= 37 -> fast slab) and
    # accumulator scales straddling the per-slab limit (|E| <= 91), plus growth
    # within a slab: the fast path, the generic slab and the thread recompute
    # must all give the oracle's bits
    rng = np.random.default_rng(abs(ea) * 1000 + abs(ec))
    k = 48
    A = np.ldexp(rng.uniform(1.0, 2.0, (m, k)) * rng.choice([-1.0, 1.0], (m, k)), ea + rng.integers(-2, 3, (m, k)))
    B = np.ldexp(rng.uniform(1.0, 2.0, (k, n)) * rng.choice([-1.0, 1.0], (k, n)), ea + rng.integers(-2, 3, (k, n)))
    C = np.ldexp(rng.standard_normal((m, n)), ec + rng.integers(-3, 4, (m, n)))
    A, B, C = _pats(A), _pats(B), _pats(C)
    assert mismatch(_gpu_gemm(A, B, C), O.gemm(A, B, C)) == 0


@pytest.mark.parametrize("ea", [37, -37, 35])
@pytest.mark.parametrize("m,n", [(300, 520), (520, 300), (330, 330)])
def test_gemm_tiled_product_table_edges(cuda_ok, ea, m, n):
    # shapes above the tiny-kernel cut-off, so the tiled kernels run: operand
    # scales at the staging limit (|Ea|, |Eb| = 37 -> Ea + Eb + n at the ends of
    # the PIX product table), both signs, accumulators of either sign and scale
    rng = np.random.default_rng(abs(ea) * 7 + m)
    k = 48
    A = np.ldexp(rng.uniform(1.0, 2.0, (m, k)) * rng.choice([-1.0, 1.0], (m, k)), ea + rng.integers(-1, 1, (m, k)))
    B = np.ldexp(rng.uniform(1.0, 2.0, (k, n)) * rng.choice([-1.0, 1.0], (k, n)), ea + rng.integers(-1, 1, (k, n)))
    C = np.ldexp(rng.standard_normal((m, n)), 2 * ea + rng.integers(-2, 3, (m, n)))
    A, B, C = _pats(A), _pats(B), _pats(C)
    assert mismatch(_gpu_gemm(A, B, C), O.gemm(A, B, C)) == 0


@pytest.mark.parametrize("ea", [37, -37])
def test_syrk_tiled_product_table_edges(cuda_ok, ea):
    import paper_2401_14117_b200 as PB
    rng = np.random.default_rng(abs(ea) + 11)
    n, k = 330, 40
    A = np.ldexp(rng.uniform(1.0, 2.0, (n, k)) * rng.choice([-1.0, 1.0], (n, k)), ea + rng.integers(-1, 1, (n, k)))
    C = np.ldexp(rng.standard_normal((n, n)), 2 * ea)
    A, C = _pats(A), _pats(C)
    dC = to_dev(C)
    PB.posit_syrk(to_dev(A), dC)
    assert mismatch(to_host(dC), O.syrk_lower(A, C)) == 0


@pytest.mark.parametrize("transa,transb", [("N", "N"), ("T", "N"), ("N", "T")])
@pytest.mark.parametrize("alpha,beta", [(2.5, 0.75), (-3.0, 1.0), (1.0, 0.0), (0.1, -2.0), (-1.0, 1.0)])
def test_gemm_eq2_general_alpha_beta(cuda_ok, transa, transb, alpha, beta):
    import paper_2401_14117_b200 as PB
    A, B, C = SI.config2(n=130, m=70, k=45)
    if transa == "T":
        A = A.T.copy()
    if transb == "T":
        B = B.T.copy()
    A, B, C = _pats(A), _pats(B), _pats(C)
    a, b = O.from_f64(alpha), O.from_f64(beta)
    dC = to_dev(C)
    PB.posit_gemm_eq2(to_dev(A), to_dev(B), dC, a, b, transb=transb, transa=transa)
    assert mismatch(to_host(dC), O.gemm_eq2(A, B, C, a, b, transa=transa, transb=transb)) == 0


@pytest.mark.parametrize("transb", ["N", "T"])
@pytest.mark.parametrize("beta", [ONE, 0])
def test_gemm_host_pipelined_matches_oracle(cuda_ok, transb, beta):
    # posit_gemm_host with m >= 1024 takes the chunked, stream-pipelined schedule
    # (two row chunks here: 576 rows and a ragged 524); sampled rows around the
    # chunk boundary are checked against the oracle, all of C against the device GEMM.
    import os
    import torch
    import paper_2401_14117_b200 as PB
    m, n, k = 1100, 96, 70
    A64, B64, C64 = SI.config2(n=n, m=m, k=k)
    if transb == "T":
        B64 = B64.T.copy()
    A, B, C = _pats(A64), _pats(B64), _pats(C64)
    h = [torch.from_numpy(x.view(np.int32)).pin_memory() for x in (A, B, C)]
    dwork = torch.empty(PB.posit_gemm_host_work_bytes(m, n, k), dtype=torch.uint8, device="cuda")
    PB.posit_gemm_host(h[0], h[1], h[2], dwork, transb=transb, beta=beta)
    got = h[2].numpy().view(np.uint32).copy()
    rows = np.r_[0:3, 570:582, 1090:1100]
    ref = O.gemm(A[rows], B, C[rows] if beta else np.zeros_like(C[rows]), transb=transb, beta=beta)
    assert mismatch(got[rows], ref) == 0
    dev = _gpu_gemm(A, B, C, transb=transb, beta=beta)
    assert mismatch(got, dev) == 0


@pytest.mark.parametrize("transa", ["N", "T"])
@pytest.mark.parametrize("transb", ["N", "T"])
@pytest.mark.parametrize("alpha,beta", [(MONE, ONE), (ONE, 0)])
def test_gemm_tiny_path_special_values(cuda_ok, transa, transb, alpha, beta):
    # m, n <= 128 and K <= 64 run the one-thread-per-output kernel (the panel-
    # internal updates); zeros, NaR, extreme scales and accumulators beyond the
    # fast range force its generic fallback on some elements
    m, n, k = 60, 100, 40
    A = _pats(SI.normal_matrix((m, k), 1.0, 21))
    B = _pats(SI.normal_matrix((k, n), 1e3, 22))
    C = _pats(SI.normal_matrix((m, n), 1e20, 23))
    A[5, 7] = O.P32_NAR
    A[9, :] = 0
    A[11, 3] = O.from_f64(1e30)
    B[12, 40] = O.from_f64(1e-33)
    C[:, 0] = O.from_f64(2.0 ** 110)
    if transa == "T":
        A = A.T.copy()
    if transb == "T":
        B = B.T.copy()
    ref = O.gemm(A, B, C, transa=transa, transb=transb, alpha=alpha, beta=beta)
    assert mismatch(_gpu_gemm(A, B, C, transb, alpha=alpha, beta=beta, transa=transa), ref) == 0


def test_accumulator_encode_exhaustive_identity(cuda_ok):
    # C <- C (-) 0 (x) B over all 2^32 patterns of C: every output goes through
    # the accumulator decode and the exact lattice encoder (acc_encode) and must
    # come back bit for bit (NaR stays NaR)
    import torch
    import paper_2401_14117_b200 as PB
    side = 8192
    A = torch.zeros(side, 1, dtype=torch.int32, device="cuda")
    B = torch.full((1, side), 0x40000000, dtype=torch.int32, device="cuda")
    bad = 0
    for c0 in range(0, 1 << 32, side * side):
        C0 = torch.arange(c0, c0 + side * side, dtype=torch.int64, device="cuda").to(torch.int32).view(side, side)
        C = C0.clone()
        PB.posit_gemm(A, B, C)
        bad += int((C != C0).sum())
        del C0, C
    assert bad == 0
