"""The multi-GPU LU schedule (paper_2401_14117_b200/dist.py) on CPU: gloo
process groups of world size 2 and 3, the arithmetic supplied by the oracle
(test infrastructure) through the same five-call ``ops`` interface the CUDA
path implements.  The gathered factors, ipiv and info must equal the textbook
unblocked oracle LU bit for bit (Q6: distribution is a traversal
change only), for every P.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic_inputs as SI
from oracle import oracle as O
from paper_2401_14117_b200.dist import BlockCyclic1D, getrf_dist


def _np(t):
    return t.contiguous().numpy().view(np.uint32)


class OracleOps:
    """CPU stand-in for CudaOps (tests only)."""

    def getrf_panel(self, P, ipiv, info, row_base):
        lu, piv, inf = O.getrf(_np(P))
        P.copy_(torch.from_numpy(lu.view(np.int32)))
        ipiv.copy_(torch.from_numpy(piv + row_base))
        if int(info[0]) == 0 and inf != 0:
            info[0] = inf + row_base

    def laswp(self, A, k1, k2, ipiv):
        for k in range(k1, k2):
            p = int(ipiv[k]) - 1
            if p != k:
                t = A[k].clone()
                A[k] = A[p]
                A[p] = t

    def trsm_llnu(self, L, B):
        if B.shape[1]:
            B.copy_(torch.from_numpy(O.trsm_llnu(_np(L), _np(B)).view(np.int32)))

    def gemm_minus(self, A, B, C):
        if C.shape[0] and C.shape[1]:
            C.copy_(torch.from_numpy(O.gemm(_np(A), _np(B), _np(C)).view(np.int32)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, nb, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = A.shape[0]
        desc = BlockCyclic1D(n, nb, world, rank)
        full = torch.from_numpy(A.view(np.int32))
        loc = desc.scatter(full)
        ipiv = torch.zeros(n, dtype=torch.int32)
        info = torch.zeros(1, dtype=torch.int32)
        getrf_dist(loc, desc, ipiv, info, ops=OracleOps())
        out[rank] = (loc.numpy().copy(), ipiv.numpy().copy(), int(info[0]))
    finally:
        dist.destroy_process_group()


def _run(A, nb, world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), A, nb, out), nprocs=world, join=True)
    n = A.shape[0]
    desc = BlockCyclic1D(n, nb, world, 0)
    full = desc.gather([torch.from_numpy(out[r][0]) for r in range(world)]).numpy().view(np.uint32)
    return full, [out[r][1] for r in range(world)], [out[r][2] for r in range(world)]


def test_block_cyclic_descriptor():
    d = BlockCyclic1D(100, 16, 3, 1)
    assert d.nblocks == 7 and d.local_blocks() == [1, 4] and d.local_cols() == 32
    assert BlockCyclic1D(100, 16, 3, 0).local_cols() == 16 + 16 + 4     # blocks 0, 3, 6 (ragged)
    assert d.local_offset(4) == 16 and d.first_local_after(1) == 16 and d.first_local_after(4) == 32
    A = torch.arange(100 * 100, dtype=torch.int32).view(100, 100)
    parts = [BlockCyclic1D(100, 16, 3, r).scatter(A) for r in range(3)]
    assert torch.equal(d.gather(parts), A)


@pytest.mark.parametrize("world,n,nb", [(2, 80, 16), (3, 70, 8)])
def test_getrf_dist_gloo_matches_oracle(world, n, nb):
    A = O.from_f64_array(SI.config4(n))           # configs[3] recipe (U[-1,1), seed 3) at small n
    full, pivs, infos = _run(A, nb, world)
    ref, rpiv, rinfo = O.getrf(A)
    assert int(np.count_nonzero(full != ref)) == 0
    for p, i in zip(pivs, infos):
        assert np.array_equal(p, rpiv) and i == rinfo


def test_getrf_dist_gloo_zero_pivot_info():
    # a rank-deficient matrix: column 20 equals column 3 -> an exact zero pivot appears
    n, nb = 48, 8
    A64 = SI.config4(n)
    A64[:, 20] = 0.0
    A = O.from_f64_array(A64)
    full, pivs, infos = _run(A, nb, 2)
    ref, rpiv, rinfo = O.getrf(A)
    assert rinfo == 21
    assert int(np.count_nonzero(full != ref)) == 0 and all(i == rinfo for i in infos)


# ------------------------------------------------------------- Cholesky ------
from paper_2401_14117_b200.dist import potrf_dist  # noqa: E402


class OracleCholOps:
    """CPU stand-in for CudaCholOps (tests only)."""

    def potrf_block(self, D, info, row_base):
        l, inf = O.potrf_lower(_np(D))
        D.copy_(torch.from_numpy(l.view(np.int32)))
        if int(info[0]) == 0 and inf != 0:
            info[0] = inf + row_base

    def trsm_rltn(self, L, B):
        if B.shape[0]:
            B.copy_(torch.from_numpy(O.trsm_rltn(_np(L), _np(B)).view(np.int32)))

    def syrk_minus(self, A, C):
        if C.shape[0]:
            C.copy_(torch.from_numpy(O.syrk_lower(_np(A), _np(C)).view(np.int32)))

    def gemm_nt_minus(self, A, B, C):
        if C.shape[0] and C.shape[1]:
            C.copy_(torch.from_numpy(O.gemm(_np(A), _np(B), _np(C), transb="T").view(np.int32)))


def _chol_worker(rank, world, port, A, nb, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = A.shape[0]
        desc = BlockCyclic1D(n, nb, world, rank)
        loc = desc.scatter(torch.from_numpy(A.view(np.int32)))
        info = torch.zeros(1, dtype=torch.int32)
        potrf_dist(loc, desc, info, ops=OracleCholOps())
        out[rank] = (loc.numpy().copy(), int(info[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,nb", [(2, 72, 16), (3, 61, 8)])
def test_potrf_dist_gloo_matches_oracle(world, n, nb):
    A = O.from_f64_array(SI.config3(n))           # configs[2] recipe (G G^T / n + I) at small n
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_chol_worker, args=(world, _free_port(), A, nb, out), nprocs=world, join=True)
    desc = BlockCyclic1D(n, nb, world, 0)
    full = desc.gather([torch.from_numpy(out[r][0]) for r in range(world)]).numpy().view(np.uint32)
    ref, rinfo = O.potrf_lower(A)
    il = np.tril_indices(n)
    assert rinfo == 0 and int(np.count_nonzero(full[il] != ref[il])) == 0
    assert all(out[r][1] == 0 for r in range(world))


# ------------------------------------------------------ column-split GEMM ----
from paper_2401_14117_b200.dist import col_slab, gemm_colsplit  # noqa: E402


def test_col_slab_partition():
    for n in (1, 7, 64, 100, 4096):
        for P in (1, 2, 3, 4, 8):
            cuts = [col_slab(n, P, r) for r in range(P)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            assert all(cuts[r][1] == cuts[r + 1][0] for r in range(P - 1))
            assert all(c0 % 4 == 0 or c0 == n for c0, _ in cuts)


def _gemm_worker(rank, world, port, A, B, C, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c0, c1 = col_slab(B.shape[1], world, rank)
        # only rank 0 holds A; the others receive it through the broadcast
        dA = torch.from_numpy(A.view(np.int32)).clone() if rank == 0 else torch.zeros(A.shape, dtype=torch.int32)
        Bl = torch.from_numpy(B[:, c0:c1].copy().view(np.int32))
        Cl = torch.from_numpy(C[:, c0:c1].copy().view(np.int32))
        gemm_colsplit(dA, Bl, Cl, src=0, ops=OracleOps())
        out[rank] = (c0, c1, Cl.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,k", [(2, 24, 40, 33), (3, 17, 29, 20)])
def test_gemm_colsplit_gloo_matches_oracle(world, m, n, k):
    A64, B64, C64 = SI.config2(n=n, m=m, k=k)      # configs[1] recipe at small size, ragged slabs
    A, B, C = O.from_f64_array(A64), O.from_f64_array(B64), O.from_f64_array(C64)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gemm_worker, args=(world, _free_port(), A, B, C, out), nprocs=world, join=True)
    got = np.empty_like(C)
    for r in range(world):
        c0, c1, Cl = out[r]
        got[:, c0:c1] = Cl.view(np.uint32)
    assert int(np.count_nonzero(got != O.gemm(A, B, C))) == 0
