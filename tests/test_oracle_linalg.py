"""Pins of the oracle's GEMM / SYRK / TRSM / LU / Cholesky against closed
forms, the spec's worked examples, exact special cases, binary64 residuals and
the order contract (reading Q6).

Citations: P:n = PAPER.md line n; S:n = SPEC.md line n.
"""
import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import checker as X
from oracle import oracle as O

ONE, MONE = O.P32_ONE, O.P32_MONE


def P(x):
    return O.from_f64_array(np.asarray(x, dtype=np.float64))


def F(p):
    return O.to_f64_array(p)


# ------------------------------------------------------------------ GEMM -----
def test_gemm_spec_2x2():
    # [[1,2],[3,4]] . [[5,6],[7,8]] = [[19,22],[43,50]]  (alpha=1, beta=0)
    C = O.gemm(P([[1, 2], [3, 4]]), P([[5, 6], [7, 8]]), None, alpha=ONE, beta=0)
    assert np.array_equal(F(C), [[19, 22], [43, 50]])


def test_gemm_integer_special_case_is_exact():
    # entries in {-8..8}, K = 4096: all partial sums |.| < 2^23 where
    # Posit(32,2) holds every integer exactly, so C - A.B must equal the int64 result.
    rng = np.random.default_rng(5)
    m, n, k = 6, 5, 4096
    A = rng.integers(-8, 9, (m, k))
    B = rng.integers(-8, 9, (k, n))
    C = rng.integers(-1000, 1001, (m, n))
    got = O.gemm(P(A), P(B), P(C))
    assert np.array_equal(F(got), (C - A @ B).astype(np.float64))
    for ta, tb in (("T", "N"), ("N", "T"), ("T", "T")):
        Ao = A.T.copy() if ta == "T" else A
        Bo = B.T.copy() if tb == "T" else B
        got = O.gemm(P(Ao), P(Bo), P(C), transa=ta, transb=tb, alpha=ONE)
        assert np.array_equal(F(got), (C + A @ B).astype(np.float64))


def test_gemm_matches_checker_triple_loop():
    # equals the naive fixed-order triple loop, here evaluated with the
    # independent exact-rational checker ops
    rng = np.random.default_rng(9)
    A = P(rng.standard_normal((3, 7)) * 3)
    B = P(rng.standard_normal((7, 4)) / 5)
    C = P(rng.standard_normal((3, 4)) * 40)
    got = O.gemm(A, B, C)
    for i in range(3):
        for j in range(4):
            c = int(C[i, j])
            for l in range(7):
                c = X.sub(c, X.mul(int(A[i, l]), int(B[l, j])))
            assert c == got[i, j]


def test_gemm_identity_and_bad_args():
    rng = np.random.default_rng(1)
    B = P(rng.standard_normal((8, 8)))
    C = P(rng.standard_normal((8, 8)))
    got = O.gemm(P(np.eye(8)), B, C)
    assert np.array_equal(got, O.vec_op("sub", C, B))          # exact: C (-) B
    assert np.array_equal(O.gemm(P(np.eye(8)), B, None, alpha=ONE, beta=0), B)
    with pytest.raises(ValueError):
        O.gemm(B, B, C, alpha=O.from_f64(2.0))
    with pytest.raises(ValueError):
        O.gemm(B, B, C, beta=O.from_f64(0.5))


def test_gemm_nar_propagates_to_row_and_column():
    # a NaR in A poisons exactly its output row
    rng = np.random.default_rng(2)
    A = P(rng.standard_normal((5, 6)))
    A[2, 3] = O.P32_NAR
    got = O.gemm(A, P(rng.standard_normal((6, 4))), P(rng.standard_normal((5, 4))))
    assert np.all(got[2] == O.P32_NAR) and not np.any(np.delete(got, 2, axis=0) == O.P32_NAR)


def test_syrk_equals_gemm_nt_lower_and_keeps_upper():
    rng = np.random.default_rng(3)
    A = P(rng.standard_normal((9, 13)))
    C = P(rng.standard_normal((9, 9)) * 4)
    got = O.syrk_lower(A, C)
    ref = O.gemm(A, A, C, transb="T")
    il = np.tril_indices(9)
    iu = np.triu_indices(9, 1)
    assert np.array_equal(got[il], ref[il]) and np.array_equal(got[iu], C[iu])


# ------------------------------------------------------------------ TRSM -----
def test_trsm_spec_examples():
    # diag(2,4), b = [2,4] -> [1,1]  (right / transposed non-unit variant)
    assert np.array_equal(F(O.trsm_rltn(P(np.diag([2.0, 4.0])), P([[2.0, 4.0]]))), [[1.0, 1.0]])
    # unit lower identity -> B unchanged
    B = P(np.random.default_rng(4).standard_normal((5, 3)))
    assert np.array_equal(O.trsm_llnu(P(np.eye(5)), B), B)


def test_trsm_dyadic_exact():
    # L unit lower with entries in {0, +-1/2, +-1/4}; X small integers: B = L X exactly,
    # forward substitution must return X bit-exactly
    rng = np.random.default_rng(6)
    n = 12
    L = np.tril(rng.choice([0.0, 0.5, -0.5, 0.25, -0.25], (n, n)), -1) + np.eye(n)
    Xs = rng.integers(-20, 21, (n, 4)).astype(np.float64)
    assert np.array_equal(F(O.trsm_llnu(P(L), P(L @ Xs))), Xs)
    D = np.diag([2.0 ** (i % 3) for i in range(n)])
    Lnd = L @ D                                           # non-unit lower, power-of-2 diagonal
    Y = rng.integers(-20, 21, (3, n)).astype(np.float64) * 4
    assert np.array_equal(F(O.trsm_rltn(P(Lnd), P(Y @ Lnd.T))), Y)


# -------------------------------------------------------------------- LU -----
def test_getrf_spec_example_and_identity():
    # [[0,1],[2,3]] -> ipiv [2,2], U = [[2,3],[0,1]], L21 = 0
    LU, ipiv, info = O.getrf(P([[0.0, 1.0], [2.0, 3.0]]))
    assert list(ipiv) == [2, 2] and info == 0
    assert np.array_equal(F(LU), [[2.0, 3.0], [0.0, 1.0]])
    LU, ipiv, info = O.getrf(P(np.eye(7)))
    assert np.array_equal(F(LU), np.eye(7)) and list(ipiv) == list(range(1, 8)) and info == 0


def _dyadic_lu(n, seed):
    rng = np.random.default_rng(seed)
    L = np.tril(rng.choice([0.0, 0.5, -0.5, 0.25, -0.25], (n, n)), -1) + np.eye(n)
    U = np.triu(rng.integers(-6, 7, (n, n)).astype(np.float64), 1) + np.diag(rng.choice([8.0, -8.0, 16.0], n))
    return L, U


def test_getrf_dyadic_exact():
    # |l_ik| <= 1/2 < 1 so no row swaps; every intermediate is a small dyadic -> exact
    L, U = _dyadic_lu(24, 8)
    LU, ipiv, info = O.getrf(P(L @ U))
    assert info == 0 and list(ipiv) == list(range(1, 25))
    assert np.array_equal(F(LU), np.tril(L, -1) + U)


def _lu_residual(A64, LU, ipiv):
    n = A64.shape[0]
    LUf = F(LU)
    L = np.tril(LUf, -1) + np.eye(n)
    U = np.triu(LUf)
    PA = A64.copy()
    for k, p in enumerate(ipiv):
        PA[[k, p - 1]] = PA[[p - 1, k]]
    return np.linalg.norm(PA - L @ U) / np.linalg.norm(A64)


def test_getrf_residual_config1_recipe():
    # ||PA - LU||_F / ||A||_F < 1e-6 at N = 256 (config 1 recipe, U[-1,1) seed 0)
    A64 = F(P(SI.config1()))
    LU, ipiv, info = O.getrf(P(A64))
    assert info == 0
    assert _lu_residual(A64, LU, ipiv) < 1e-6
    assert np.all(ipiv >= np.arange(1, 257))


def blocked_getrf_from_oracle_pieces(A, nb):
    """Right-looking blocked LU composed from oracle pieces (panel getrf, laswp,
    trsm_llnu, gemm C -= A B): a traversal change only under the order contract."""
    A = A.copy()
    n = A.shape[0]
    ipiv = np.zeros(n, np.int32)
    info = 0
    for s in range(0, n, nb):
        b = min(nb, n - s)
        panel, piv, pinfo = O.getrf(A[s:, s:s + b])
        A[s:, s:s + b] = panel
        if pinfo and not info:
            info = s + pinfo
        for k in range(b):
            ipiv[s + k] = s + piv[k]
            r0, r1 = s + k, s + piv[k] - 1
            if r0 != r1:
                for cols in (slice(0, s), slice(s + b, n)):
                    tmp = A[r0, cols].copy()
                    A[r0, cols] = A[r1, cols]
                    A[r1, cols] = tmp
        if s + b < n:
            A[s:s + b, s + b:] = O.trsm_llnu(A[s:s + b, s:s + b], A[s:s + b, s + b:])
            A[s + b:, s + b:] = O.gemm(A[s + b:, s:s + b], A[s:s + b, s + b:], A[s + b:, s + b:])
    return A, ipiv, info


def test_getrf_block_size_invariance():
    # under c <- c (-) a (x) b ascending k, blocking changes nothing
    A = P(SI.lu_matrix(40, seed=12))
    ref, rpiv, rinfo = O.getrf(A)
    for nb in (1, 3, 8, 32):
        got, piv, info = blocked_getrf_from_oracle_pieces(A, nb)
        assert np.array_equal(got, ref) and np.array_equal(piv, rpiv) and info == rinfo


def test_getrf_zero_pivot_info():
    # Q11: first zero column -> info (1-based), factorisation continues
    A = SI.lu_matrix(6, seed=3)
    A[:, 2] = 0.0
    LU, ipiv, info = O.getrf(P(A))
    assert info == 3


# -------------------------------------------------------------- Cholesky -----
def test_potrf_spec_examples():
    L, info = O.potrf_lower(P(np.diag([4.0, 9.0])))
    assert info == 0 and np.array_equal(F(L), np.diag([2.0, 3.0]))
    L, info = O.potrf_lower(P(np.eye(6)))
    assert info == 0 and np.array_equal(F(L), np.eye(6))


def test_potrf_dyadic_exact_and_upper_untouched():
    rng = np.random.default_rng(10)
    n = 16
    L = np.tril(rng.choice([0.0, 0.5, -0.5, 0.25, 1.0, -1.0], (n, n)), -1) + np.diag(rng.choice([4.0, 16.0, 8.0 * 2], n))
    A = L @ L.T
    Ap = P(A)
    Ap[np.triu_indices(n, 1)] = 0x12345678               # upper must not be read or written
    got, info = O.potrf_lower(Ap)
    assert info == 0
    assert np.array_equal(F(np.tril(got)), L)
    assert np.all(got[np.triu_indices(n, 1)] == 0x12345678)


def test_potrf_not_pd_info():
    A = np.diag([4.0, 9.0, -1.0, 4.0])
    _, info = O.potrf_lower(P(A))
    assert info == 3


def test_potrf_residual_config3_recipe_small():
    A64 = F(P(SI.config3(128)))
    L, info = O.potrf_lower(P(A64))
    assert info == 0
    Lf = np.tril(F(L))
    assert np.linalg.norm(A64 - Lf @ Lf.T) / np.linalg.norm(A64) < 1e-6


def blocked_potrf_from_oracle_pieces(A, nb):
    A = A.copy()
    n = A.shape[0]
    for s in range(0, n, nb):
        b = min(nb, n - s)
        blk, info = O.potrf_lower(A[s:s + b, s:s + b])
        A[s:s + b, s:s + b] = np.where(np.tril(np.ones((b, b), bool)), blk, A[s:s + b, s:s + b])
        if info:
            return A, s + info
        if s + b < n:
            A[s + b:, s:s + b] = O.trsm_rltn(A[s:s + b, s:s + b], A[s + b:, s:s + b])
            A[s + b:, s + b:] = O.syrk_lower(A[s + b:, s:s + b], A[s + b:, s + b:])
    return A, 0


def test_potrf_block_size_invariance():
    A = P(SI.config3(36))
    ref, rinfo = O.potrf_lower(A)
    for nb in (1, 5, 8, 32):
        got, info = blocked_potrf_from_oracle_pieces(A, nb)
        assert info == rinfo == 0
        assert np.array_equal(np.tril(got), np.tril(ref))


# ------------------------------------------------------------- solves -----
# Rgetrs / Rpotrs of the accuracy study, reading Q21: reference
# BLAS trsv loop order (forward: ascending k; back: descending k).
def test_getrs_potrs_spec_examples():
    b = P([4.0, 9.0])
    L, info = O.potrf_lower(P(np.diag([4.0, 9.0])))
    assert info == 0 and np.array_equal(F(O.potrs_lower(L, b)), [1.0, 1.0])
    bb = P(SI.normal_matrix((6,), 1.0, 3))
    assert np.array_equal(O.potrs_lower(P(np.eye(6)), bb), bb)                    # S:239 (L = I)
    LU, ipiv, info = O.getrf(P(np.eye(6)))
    assert np.array_equal(O.getrs(LU, ipiv, bb), bb)


def test_getrs_dyadic_exact_with_pivots():
    # P A = L U with dyadic L, U and an explicit row permutation; x small integers:
    # every intermediate of both substitutions is exact, so x is recovered exactly
    n = 16
    L, U = _dyadic_lu(n, 21)
    perm = np.random.default_rng(4).permutation(n)
    A = (L @ U)[np.argsort(perm)]            # rows permuted: getrf must undo it
    x = np.random.default_rng(5).integers(-4, 5, n).astype(np.float64)
    LU, ipiv, info = O.getrf(P(A))
    assert info == 0
    got = F(O.getrs(LU, ipiv, P(A @ x)))
    assert np.array_equal(got, x), (got, x)         # every intermediate exact: x recovered bit for bit


def _checker_back_desc(U, y):
    # brute force with exact-rational ops in the Q21 order (descending k)
    n = len(y)
    y = [int(v) for v in y]
    for i in range(n - 1, -1, -1):
        for k in range(n - 1, i, -1):
            y[i] = X.sub(y[i], X.mul(int(U[i, k]), y[k]))
        y[i] = X.div(y[i], int(U[i, i]))
    return y


def _checker_fwd(L, b, unit):
    n = len(b)
    b = [int(v) for v in b]
    for i in range(n):
        for k in range(i):
            b[i] = X.sub(b[i], X.mul(int(L[i, k]), b[k]))
        if not unit:
            b[i] = X.div(b[i], int(L[i, i]))
    return b


def test_getrs_potrs_match_checker_brute_force():
    n = 7
    A = P(SI.lu_matrix(n, 11))
    b = P(SI.normal_matrix((n,), 1.0, 12))
    LU, ipiv, _ = O.getrf(A)
    pb = [int(v) for v in b]
    for k, p in enumerate(ipiv):
        pb[k], pb[p - 1] = pb[p - 1], pb[k]
    y = _checker_fwd(LU, pb, unit=True)
    assert list(O.getrs(LU, ipiv, b)) == _checker_back_desc(LU, y)
    S = P(SI.config3(n))
    Lc, _ = O.potrf_lower(S)
    y = _checker_fwd(Lc, b, unit=False)
    assert list(O.potrs_lower(Lc, b)) == _checker_back_desc(Lc.T.copy(), y)


def test_gemm_eq2_general_alpha_beta_vs_checker():
    # Eq.2 in SPEC S:200's order, brute force with exact-rational ops
    rng = np.random.default_rng(77)
    m, n, k = 3, 4, 5
    A = P(rng.standard_normal((m, k)))
    B = P(rng.standard_normal((k, n)))
    C = P(rng.standard_normal((m, n)))
    for alpha, beta in [(2.5, 0.75), (-3.0, 1.0), (1.0, 0.0), (0.1, -2.0)]:
        a, b = O.from_f64(alpha), O.from_f64(beta)
        got = O.gemm_eq2(A, B, C, a, b)
        for i in range(m):
            for j in range(n):
                t = 0
                for l in range(k):
                    t = X.add(t, X.mul(int(A[i, l]), int(B[l, j])))
                assert int(got[i, j]) == X.add(X.mul(a, t), X.mul(b, int(C[i, j])))
    # alpha = 1, beta = 0 -> the plain product
    got = O.gemm_eq2(P([[1.0, 2.0], [3.0, 4.0]]), P([[5.0, 6.0], [7.0, 8.0]]), np.zeros((2, 2), np.uint32), ONE, 0)
    assert np.array_equal(F(got), [[19.0, 22.0], [43.0, 50.0]])
