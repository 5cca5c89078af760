"""Full-size (BASELINE.json configs, the sizes bench.py times) parity by
properties that hold at any size and by leading-column slabs the oracle can
compute exactly:

* left-looking slab property: columns 0..k-1 of the LU (L below, U above the
  diagonal) and ipiv[0:k] depend only on A[:, 0:k], so the oracle's getrf on
  the n x k slab must match the GPU factors of the full matrix bit for bit
  (same for Cholesky with potrf(A11) + trsm on the n x k lower slab);
* block-size invariance (reading Q6): nb = 256 and nb = 96 give identical bits;
* binary64 residual ||PA - LU||_F / ||A||_F (resp. ||A - LL^T||) within
  n * 2^-27 (f_s = 27 near 1), evaluated on the GPU in binary64.
"""
import numpy as np
import pytest
import torch

import synthetic_inputs as SI
from oracle import oracle as O
from tests.gpu_util import mismatch

pytestmark = pytest.mark.gpu

K_SLAB = 48


def _lu_gpu(A64, nb):
    import paper_2401_14117_b200 as PB
    n = A64.shape[0]
    dA = PB.posit_from_f64(torch.from_numpy(A64).cuda())
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    PB.posit_getrf(dA, ipiv, info, nb=nb)
    return dA, ipiv, int(info.cpu()[0])


def _lu_residual_gpu(A64, dLU, ipiv):
    import paper_2401_14117_b200 as PB
    n = A64.shape[0]
    LU = PB.posit_to_f64(dLU)
    L = torch.tril(LU, -1) + torch.eye(n, dtype=torch.float64, device="cuda")
    U = torch.triu(LU)
    A = torch.from_numpy(A64).cuda()
    perm = torch.arange(n, device="cuda")
    piv = ipiv.cpu().numpy() - 1
    p = perm.cpu().numpy()
    for k in range(n):                      # compose the row interchanges
        p[[k, piv[k]]] = p[[piv[k], k]]
    PA = A[torch.from_numpy(p).cuda()]
    return float(torch.linalg.norm(PA - L @ U) / torch.linalg.norm(A))


@pytest.mark.parametrize("cfg", ["C4", "C5m16", "C5p16"])
def test_lu_full_size_slab_residual_and_block_invariance(cuda_ok, cfg):
    if cfg == "C4":
        A64, nb = SI.config4(), SI.C4_NB
    else:
        A64, nb = SI.config5(-16 if cfg == "C5m16" else 16), SI.C5_NB
    n = A64.shape[0]
    dLU, ipiv, info = _lu_gpu(A64, nb)
    got = dLU.cpu().numpy().view(np.uint32)
    # slab: the oracle factors A[:, :k] (n x k); the later steps' row
    # interchanges (ipiv[k:]) then permute rows >= k of those columns
    Ap = O.from_f64_array(A64[:, :K_SLAB])
    ref, rpiv, rinfo = O.getrf(Ap)
    gpiv = ipiv.cpu().numpy()
    assert np.array_equal(gpiv[:K_SLAB], rpiv)
    for k in range(K_SLAB, n):
        p = gpiv[k] - 1
        if p != k:
            ref[[k, p]] = ref[[p, k]]
    assert mismatch(got[:, :K_SLAB], ref) == 0
    assert info == 0 and rinfo == 0
    # U's first k rows: U12 = L11^-1 (P_k A)[:k, k:] by the oracle's TRSM
    Pk = O.from_f64_array(A64[:, K_SLAB:])
    for k in range(K_SLAB):
        p = gpiv[k] - 1
        if p != k:
            Pk[[k, p]] = Pk[[p, k]]
    L11 = np.tril(ref[:K_SLAB, :K_SLAB], -1) | np.diag(np.full(K_SLAB, O.P32_ONE, np.uint32))
    U12 = O.trsm_llnu(L11, Pk[:K_SLAB].copy())
    assert mismatch(got[:K_SLAB, K_SLAB:], U12) == 0
    # residual in binary64 on the GPU
    assert _lu_residual_gpu(A64, dLU, ipiv) < n * 2.0 ** -27
    # block-size invariance at full size
    dLU2, ipiv2, _ = _lu_gpu(A64, 96)
    assert torch.equal(dLU, dLU2) and torch.equal(ipiv, ipiv2)


def test_cholesky_config3_full_size(cuda_ok):
    import paper_2401_14117_b200 as PB
    A64 = SI.config3()
    n = A64.shape[0]
    dA = PB.posit_from_f64(torch.from_numpy(A64).cuda())
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    PB.posit_potrf(dA, info, nb=SI.C3_NB)
    assert int(info.cpu()[0]) == 0
    got = dA.cpu().numpy().view(np.uint32)
    # slab: L[:, :k] = potrf(A11) and A21 L11^-T, by the oracle
    Ap = O.from_f64_array(A64[:, :K_SLAB])
    L11, rinfo = O.potrf_lower(Ap[:K_SLAB].copy())
    L21 = O.trsm_rltn(L11, Ap[K_SLAB:].copy())
    il = np.tril_indices(K_SLAB)
    assert rinfo == 0 and mismatch(got[:K_SLAB, :K_SLAB][il], L11[il]) == 0
    assert mismatch(got[K_SLAB:, :K_SLAB], L21) == 0
    # residual ||A - L L^T|| / ||A|| in binary64 on the GPU
    L = torch.tril(PB.posit_to_f64(dA))
    A = torch.from_numpy(A64).cuda()
    assert float(torch.linalg.norm(A - L @ L.T) / torch.linalg.norm(A)) < n * 2.0 ** -27
    # block-size invariance
    dB = PB.posit_from_f64(torch.from_numpy(A64).cuda())
    PB.posit_potrf(dB, info, nb=128)
    assert torch.equal(torch.tril(dA), torch.tril(dB))
