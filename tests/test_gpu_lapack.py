"""GPU parity of posit_trsm / posit_getrf / posit_potrf with the CPU oracle
(textbook unblocked loops), bit-exact on every output word, ipiv and info."""
import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import oracle as O
from tests.gpu_util import mismatch, to_dev, to_host

pytestmark = pytest.mark.gpu


def _pats(x):
    return O.from_f64_array(x)


def _gpu_getrf(A, nb):
    import torch
    import paper_2401_14117_b200 as PB
    dA = to_dev(A)
    m, n = A.shape
    ipiv = torch.zeros(min(m, n), dtype=torch.int32, device="cuda")
    info = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    PB.posit_getrf(dA, ipiv, info, nb=nb)
    return to_host(dA), ipiv.cpu().numpy(), int(info.cpu()[0])


def _gpu_potrf(A, nb):
    import torch
    import paper_2401_14117_b200 as PB
    dA = to_dev(A)
    info = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    PB.posit_potrf(dA, info, nb=nb)
    return to_host(dA), int(info.cpu()[0])


def test_trsm_llnu_matches_oracle(cuda_ok):
    import paper_2401_14117_b200 as PB
    for m, n in [(1, 5), (37, 100), (33, 65), (256, 300), (256, 1000)]:
        L = _pats(np.tril(SI.lu_matrix(m, 1), -1) + np.eye(m))
        B = _pats(SI.normal_matrix((m, n), 1.0, 2))
        dB = to_dev(B)
        PB.posit_trsm("L", "L", "N", "U", to_dev(L), dB)
        assert mismatch(to_host(dB), O.trsm_llnu(L, B)) == 0


def test_trsm_rltn_matches_oracle(cuda_ok):
    import paper_2401_14117_b200 as PB
    for m, n in [(5, 1), (100, 37), (300, 256)]:
        L = _pats(np.tril(SI.lu_matrix(n, 1), -1) + np.diag(1.0 + np.arange(n) % 3))
        B = _pats(SI.normal_matrix((m, n), 1.0, 2))
        dB = to_dev(B)
        PB.posit_trsm("R", "L", "T", "N", to_dev(L), dB)
        assert mismatch(to_host(dB), O.trsm_rltn(L, B)) == 0


@pytest.mark.parametrize("m,n", [(1, 1), (33, 17), (75, 200), (97, 256), (64, 255)])
def test_trsm_rltn_d_fast_slow_transitions(cuda_ok, m, n):
    # the element-right-looking D-MAC kernel (k_trsm_rltn_d, n <= 256): rows
    # scaled by 2^-s_r and a tiny diagonal entry at column n // 2 make the
    # quotient leave the fast range at that step for some warps only (the
    # generic path then finishes those rows from the same state); an exact
    # zero below the diagonal at column 3n // 4 sends every warp to the
    # generic path there; ragged m and n leave partial CTAs and column groups
    import paper_2401_14117_b200 as PB
    L64 = np.tril(SI.lu_matrix(n, 21), -1) + np.diag(1.0 + np.arange(n) % 3)
    if n > 4:
        L64[n // 2, n // 2] = 2.0 ** -45
        L64[n - 1, (3 * n) // 4] = 0.0
    s = np.random.default_rng(22).integers(0, 20, m)
    B64 = SI.normal_matrix((m, n), 1.0, 23) * np.ldexp(1.0, -s)[:, None]
    L, B = _pats(L64), _pats(B64)
    dB = to_dev(B)
    PB.posit_trsm("R", "L", "T", "N", to_dev(L), dB)
    assert mismatch(to_host(dB), O.trsm_rltn(L, B)) == 0


@pytest.mark.parametrize("m,n", [(1, 1), (17, 33), (200, 75), (256, 97), (255, 64), (256, 1000)])
def test_trsm_llnu_d_fast_slow_transitions(cuda_ok, m, n):
    # the element-right-looking D-MAC kernel (k_trsm_llnu_d, m <= 256):
    # columns scaled by 2^s_c with a large entry at row m // 2 (x_k leaves the
    # fast range there for some warps only), an exact zero in L below the
    # diagonal of column 3m // 4 (every warp takes the generic path there),
    # ragged m and n (partial column groups and CTAs)
    import paper_2401_14117_b200 as PB
    L64 = np.tril(SI.lu_matrix(m, 31), -1) + np.eye(m)
    if m > 4:
        L64[m - 1, (3 * m) // 4] = 0.0
    s = np.random.default_rng(32).integers(0, 20, n)
    B64 = SI.normal_matrix((m, n), 1.0, 33) * np.ldexp(1.0, s)[None, :]
    if m > 4:
        B64[m // 2, :] = np.ldexp(1.0, 25 + s)          # |E| > 37 for s > 12
    L, B = _pats(L64), _pats(B64)
    dB = to_dev(B)
    PB.posit_trsm("L", "L", "N", "U", to_dev(L), dB)
    assert mismatch(to_host(dB), O.trsm_llnu(L, B)) == 0


def test_getrf_config1_bit_exact(cuda_ok):
    # configs[0]: n = 256, nb = 32, U[-1,1) seed 0
    A = _pats(SI.config1())
    ref, rpiv, rinfo = O.getrf(A)
    got, piv, info = _gpu_getrf(A, 32)
    assert mismatch(got, ref) == 0 and np.array_equal(piv, rpiv) and info == rinfo == 0


# n <= 512: the fused tail LU (one cooperative launch); n > 512: blocked steps
# with lookahead, then the fused tail for the last <= 512 columns
@pytest.mark.parametrize("m,n,nb", [(100, 77, 16), (77, 100, 16), (300, 300, 64), (64, 64, 1), (130, 130, 256),
                                    (700, 650, 96), (650, 700, 64), (620, 620, 256), (1100, 1000, 256)])
def test_getrf_ragged_and_block_sizes(cuda_ok, m, n, nb):
    A = _pats(np.random.default_rng(m + n).uniform(-1, 1, (m, n)))
    ref, rpiv, rinfo = O.getrf(A)
    got, piv, info = _gpu_getrf(A, nb)
    assert mismatch(got, ref) == 0 and np.array_equal(piv, rpiv) and info == rinfo


def test_getrf_special_cases(cuda_ok):
    # S:231, identity, zero column (info), dyadic exact
    got, piv, info = _gpu_getrf(_pats([[0.0, 1.0], [2.0, 3.0]]), 32)
    assert list(piv) == [2, 2] and info == 0 and np.array_equal(O.to_f64_array(got), [[2, 3], [0, 1]])
    got, piv, info = _gpu_getrf(_pats(np.eye(40)), 16)
    assert np.array_equal(O.to_f64_array(got), np.eye(40)) and list(piv) == list(range(1, 41))
    A = SI.lu_matrix(50, 3)
    A[:, 20] = 0.0
    Ap = _pats(A)
    ref, rpiv, rinfo = O.getrf(Ap)
    got, piv, info = _gpu_getrf(Ap, 16)
    assert rinfo == info == 21 and mismatch(got, ref) == 0 and np.array_equal(piv, rpiv)


@pytest.mark.parametrize("zero_col", [100, 300, 650])
def test_getrf_blocked_zero_pivot_and_specials(cuda_ok, zero_col):
    # n > 512: blocked steps with lookahead (zero column inside a side-stream
    # panel, or in the fused tail), NaR / zero / extreme entries elsewhere
    n = 700
    A = SI.lu_matrix(n, 21)
    A[:, zero_col] = 0.0
    A[5, 690] = np.nan                       # NaR: absorbing once column 690 is reached (after every zero_col)
    A[400, 7] = 1e30
    A[650, 320] = 1e-30
    A[200, :] *= 2.0 ** 40
    Ap = _pats(A)
    ref, rpiv, rinfo = O.getrf(Ap)
    got, piv, info = _gpu_getrf(Ap, 64)
    assert rinfo == info == zero_col + 1
    assert mismatch(got, ref) == 0 and np.array_equal(piv, rpiv)


@pytest.mark.parametrize("s", [-16, -4, 0, 4, 16])
def test_getrf_config5_scaling_small(cuda_ok, s):
    # configs[4] recipe (U[-1,1) seed 4 scaled by 2^s) at n = 384, nb = 64
    A = _pats(np.ldexp(SI.lu_matrix(384, SI.C5_SEED), s))
    ref, rpiv, rinfo = O.getrf(A)
    got, piv, info = _gpu_getrf(A, 64)
    assert mismatch(got, ref) == 0 and np.array_equal(piv, rpiv) and info == rinfo


@pytest.mark.parametrize("n,nb", [(1, 1), (50, 16), (200, 64), (300, 256), (130, 32), (400, 64), (1100, 256)])
def test_potrf_matches_oracle(cuda_ok, n, nb):
    A = _pats(SI.config3(n))
    ref, rinfo = O.potrf_lower(A)
    got, info = _gpu_potrf(A, nb)
    il = np.tril_indices(n)
    iu = np.triu_indices(n, 1)
    assert info == rinfo == 0
    assert mismatch(got[il], ref[il]) == 0
    assert mismatch(got[iu], A[iu]) == 0           # strict upper triangle untouched


def test_potrf_not_positive_definite(cuda_ok):
    A = SI.config3(80)
    A[45, 45] = -1.0
    Ap = _pats(A)
    ref, rinfo = O.potrf_lower(Ap)
    got, info = _gpu_potrf(Ap, 16)
    assert info == rinfo == 46
    # the blocks before the failing block are fully defined and bit-identical
    assert mismatch(np.tril(got)[:, :32], np.tril(ref)[:, :32]) == 0


def test_potrf_not_positive_definite_with_lookahead(cuda_ok):
    # n >= 4 nb: side-stream panels; the failure is met inside a side-stream diagonal block
    n, nb = 400, 64
    A = SI.config3(n)
    A[250, 250] = -1.0
    Ap = _pats(A)
    ref, rinfo = O.potrf_lower(Ap)
    got, info = _gpu_potrf(Ap, nb)
    assert info == rinfo == 251
    assert mismatch(np.tril(got)[:, :192], np.tril(ref)[:, :192]) == 0


@pytest.mark.parametrize("fail_at,nb", [(0, 256), (37, 256), (250, 256), (255, 256), (100, 64), (70, 128)])
def test_potrf_not_pd_inside_cluster_block(cuda_ok, fail_at, nb):
    # the one-launch diagonal-block Cholesky (k_potf2_cluster, 32 < b <= 256) stops at
    # the failing step in every CTA: info = k + 1, and inside the failing diagonal block
    # every step before k is applied -- exactly the oracle's textbook loop there
    n = 300
    A = SI.config3(n)
    A[fail_at, fail_at] = -2.0 * abs(A[fail_at, fail_at]) - 1.0
    Ap = _pats(A)
    ref, rinfo = O.potrf_lower(Ap)
    got, info = _gpu_potrf(Ap, nb)
    assert info == rinfo == fail_at + 1
    s0 = (fail_at // nb) * nb
    s1 = min(n, s0 + nb)
    il = np.tril_indices(s1 - s0)
    assert mismatch(got[s0:s1, s0:s1][il], ref[s0:s1, s0:s1][il]) == 0
    assert mismatch(np.tril(got)[:, :s0], np.tril(ref)[:, :s0]) == 0


@pytest.mark.parametrize("n", [1, 33, 300])
def test_getrs_potrs_match_oracle(cuda_ok, n):
    import torch
    import paper_2401_14117_b200 as PB
    b = _pats(SI.normal_matrix((n,), 1.0, 7))
    LU, piv, _ = O.getrf(_pats(SI.lu_matrix(n, 9)))
    db = to_dev(b)
    PB.posit_getrs(to_dev(LU), torch.from_numpy(piv).cuda(), db)
    assert mismatch(to_host(db), O.getrs(LU, piv, b)) == 0
    L, info = O.potrf_lower(_pats(SI.config3(n)))
    assert info == 0
    db = to_dev(b)
    PB.posit_potrs(to_dev(L), db)
    assert mismatch(to_host(db), O.potrs_lower(L, b)) == 0


def test_getrs_full_size_backward_error(cuda_ok):
    # configs[3] recipe at n = 4096 on the GPU factors: relative backward error (Eq.4,
    # P:470-472) of the posit solve within the textbook gamma_n = n * eps bound,
    # eps = 2^-27 (f_s = 27 near 1); S:241's 1e-6 is for n = 64
    import torch
    import paper_2401_14117_b200 as PB
    n = 4096
    A64 = SI.config4(n)
    dA = PB.posit_from_f64(torch.from_numpy(A64).cuda())
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    PB.posit_getrf(dA, ipiv, info, nb=256)
    x_sol = np.full(n, 1.0 / np.sqrt(n))
    b64 = A64 @ x_sol
    db = PB.posit_from_f64(torch.from_numpy(b64).cuda())
    PB.posit_getrs(dA, ipiv, db)
    x = PB.posit_to_f64(db).cpu().numpy()
    e = np.linalg.norm(b64 - A64 @ x) / np.linalg.norm(b64)
    assert int(info.cpu()[0]) == 0 and e < n * 2.0 ** -27


@pytest.mark.parametrize("scale", [-90, -40, 0, 40, 90])
def test_trsm_extreme_scales_and_zeros(cuda_ok, scale):
    # magnitudes outside the decoded fast range (|E| > 37 / 75) and exact zeros
    # force the in-block kernels' generic fallback path on some lanes
    import paper_2401_14117_b200 as PB
    m, n = 70, 90
    L64 = np.tril(SI.lu_matrix(m, 13), -1) + np.eye(m)
    L64[5:9, 1:4] = 0.0
    B64 = np.ldexp(SI.normal_matrix((m, n), 1.0, 14), scale)
    B64[:, 7] = 0.0
    B64[10, :] = 0.0
    B64[12, 40] = np.nan                              # NaR: absorbing down column 40
    L, B = _pats(L64), _pats(B64)
    dB = to_dev(B)
    PB.posit_trsm("L", "L", "N", "U", to_dev(L), dB)
    assert mismatch(to_host(dB), O.trsm_llnu(L, B)) == 0
    Lr64 = np.tril(np.ldexp(SI.lu_matrix(n, 15), scale // 2), -1) + np.diag(np.ldexp(1.0 + np.arange(n) % 5, scale // 2))
    Lr64[20:25, 3:6] = 0.0
    Lr = _pats(Lr64)
    Br = _pats(np.ldexp(SI.normal_matrix((m, n), 1.0, 16), scale))
    dB = to_dev(Br)
    PB.posit_trsm("R", "L", "T", "N", to_dev(Lr), dB)
    assert mismatch(to_host(dB), O.trsm_rltn(Lr, Br)) == 0


@pytest.mark.parametrize("scale", [-100, -60, 60, 100])
def test_potrf_extreme_scales(cuda_ok, scale):
    n = 100
    A = _pats(np.ldexp(SI.config3(n), scale))
    got, ginfo = _gpu_potrf(A, 32)
    ref, rinfo = O.potrf_lower(A)
    il = np.tril_indices(n)
    assert ginfo == rinfo and mismatch(got[il], ref[il]) == 0


@pytest.mark.parametrize("ncols,k1,k2", [(1, 0, 5), (45, 3, 40), (300, 10, 300), (77, 0, 600)])
def test_laswp_sequential_semantics(cuda_ok, ncols, k1, k2):
    # pure data movement: swaps applied in order, repeated and in-block pivots
    import torch
    import paper_2401_14117_b200 as PB
    m = 900
    rng = np.random.default_rng(k2)
    A = rng.integers(0, 2 ** 32, (m, ncols), dtype=np.uint64).astype(np.uint32)
    ipiv = np.arange(1, m + 1, dtype=np.int32)
    for k in range(k1, k2):
        ipiv[k] = rng.choice([k + 1, rng.integers(k + 1, m + 1), rng.integers(k1 + 1, k2 + 1), 7 * k2 % m + 1])
    ref = A.copy()
    for k in range(k1, k2):
        p = ipiv[k] - 1
        ref[[k, p]] = ref[[p, k]]
    dA = to_dev(A)
    PB.posit_laswp(dA, k1, k2, torch.from_numpy(ipiv).cuda())
    assert mismatch(to_host(dA), ref) == 0
