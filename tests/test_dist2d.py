"""The 2D Pr x Pc block-cyclic LU (paper_2401_14117_b200/dist2d.py) on CPU:
gloo process grids 2x2 and 2x3 (and 3x1, 1x2), the oracle supplying the
arithmetic through the same ops interface the CUDA path implements.  The
gathered factors, ipiv and info must equal the textbook oracle LU bit for bit
(Q6) for every grid."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic_inputs as SI
from oracle import oracle as O
from paper_2401_14117_b200.dist2d import BlockCyclic2D, Groups, getrf_dist2d
from tests.test_dist import _free_port, _np


class OracleOps2D:
    """CPU stand-in for CudaOps2D (tests only)."""

    def iamax_key(self, col, grow, row_min, key):
        x = _np(col).astype(np.int64)
        s = np.where(x >= 2 ** 31, x - 2 ** 32, x)                       # signed pattern
        a = np.where(s < 0, -s, s)                                       # abs by negation
        a = np.where(s == -(2 ** 31), -(2 ** 31), a)                     # NaR stays the minimum
        g = grow.numpy().astype(np.int64)
        ok = g >= row_min
        if not ok.any():
            key[0] = 0
            return
        k = ((a[ok] + 2 ** 31) << 31) | ((2 ** 31 - 1) - g[ok])
        key[0] = int(k.max())

    def div_rows(self, col, v):
        if col.shape[0]:
            c = _np(col)
            col.copy_(torch.from_numpy(O.vec_op("div", c, np.full_like(c, v)).view(np.int32)))

    def rank1_minus(self, l, u, C):
        if C.shape[0] and C.shape[1]:
            C.copy_(torch.from_numpy(O.gemm(_np(l), _np(u), _np(C)).view(np.int32)))

    def trsm_llnu(self, L, B):
        if B.shape[0] and B.shape[1]:
            B.copy_(torch.from_numpy(O.trsm_llnu(_np(L), _np(B)).view(np.int32)))

    def gemm_minus(self, A, B, C):
        if C.shape[0] and C.shape[1] and A.shape[1]:
            C.copy_(torch.from_numpy(O.gemm(_np(A), _np(B), _np(C)).view(np.int32)))


def _worker(rank, world, port, A, nb, Pr, Pc, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = A.shape[0]
        pr, pc = divmod(rank, Pc)
        desc = BlockCyclic2D(n, nb, Pr, Pc, pr, pc)
        groups = Groups(Pr, Pc)
        loc = desc.scatter(torch.from_numpy(A.view(np.int32)))
        ipiv = torch.zeros(n, dtype=torch.int32)
        info = torch.zeros(1, dtype=torch.int32)
        getrf_dist2d(loc, desc, ipiv, info, groups, ops=OracleOps2D())
        out[rank] = (loc.numpy().copy(), ipiv.numpy().copy(), int(info[0]))
    finally:
        dist.destroy_process_group()


def _run(A, nb, Pr, Pc):
    world = Pr * Pc
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), A, nb, Pr, Pc, out), nprocs=world, join=True)
    desc = BlockCyclic2D(A.shape[0], nb, Pr, Pc, 0, 0)
    full = desc.gather([torch.from_numpy(out[r][0]) for r in range(world)]).numpy().view(np.uint32)
    return full, [out[r][1] for r in range(world)], [out[r][2] for r in range(world)]


def test_block_cyclic_2d_descriptor():
    d = BlockCyclic2D(50, 8, 2, 3, 1, 2)
    assert list(d.rows()[:3]) == [8, 9, 10] and d.local_row(25) == 9 and d.owner_row(25) == 1
    assert list(d.cols()[:2]) == [16, 17] and d.owner_col(45) == 2 and d.local_col(45) == 13
    A = torch.arange(50 * 50, dtype=torch.int32).view(50, 50)
    parts = [BlockCyclic2D(50, 8, 2, 3, r // 3, r % 3).scatter(A) for r in range(6)]
    assert torch.equal(d.gather(parts), A)


@pytest.mark.parametrize("Pr,Pc,n,nb", [(2, 2, 56, 8), (2, 3, 45, 8), (3, 1, 40, 8), (1, 2, 36, 8)])
def test_getrf_dist2d_gloo_matches_oracle(Pr, Pc, n, nb):
    A = O.from_f64_array(SI.config4(n))
    full, pivs, infos = _run(A, nb, Pr, Pc)
    ref, rpiv, rinfo = O.getrf(A)
    assert int(np.count_nonzero(full != ref)) == 0
    for p, i in zip(pivs, infos):
        assert np.array_equal(p, rpiv) and i == rinfo


def test_getrf_dist2d_zero_pivot():
    n, nb = 40, 8
    A64 = SI.config4(n)
    A64[:, 13] = 0.0
    A = O.from_f64_array(A64)
    full, pivs, infos = _run(A, nb, 2, 2)
    ref, rpiv, rinfo = O.getrf(A)
    assert rinfo == 14 and int(np.count_nonzero(full != ref)) == 0 and all(i == rinfo for i in infos)
