"""The distributed LU driver's CUDA path (CudaOps through the C ABI) at P = 1
on one GPU, and the block-cyclic local layout emulated for P = 2, 4 on one
device: every 'rank' is driven in lock-step by this process with the panel
'broadcast' a device copy, so no kernels wait on one another.  Bit-exact
against the textbook oracle LU (Q6)."""
import numpy as np
import pytest
import torch

import synthetic_inputs as SI
from oracle import oracle as O
from paper_2401_14117_b200.dist import BlockCyclic1D, CudaOps, getrf_dist
from tests.gpu_util import mismatch, to_dev, to_host

pytestmark = pytest.mark.gpu


def test_getrf_dist_p1_cuda(cuda_ok):
    n, nb = 300, 32
    A = O.from_f64_array(SI.config4(n))
    desc = BlockCyclic1D(n, nb, 1, 0)
    loc = desc.scatter(to_dev(A))
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    getrf_dist(loc, desc, ipiv, info)
    ref, rpiv, rinfo = O.getrf(A)
    assert mismatch(to_host(loc), ref) == 0
    assert np.array_equal(ipiv.cpu().numpy(), rpiv) and int(info.cpu()[0]) == rinfo


@pytest.mark.parametrize("P", [2, 4])
def test_getrf_dist_emulated_ranks_cuda(cuda_ok, P):
    import paper_2401_14117_b200.dist as D
    n, nb = 200, 16
    A = O.from_f64_array(SI.config4(n))
    full = to_dev(A)
    descs = [BlockCyclic1D(n, nb, P, r) for r in range(P)]
    locs = [d.scatter(full) for d in descs]
    ipivs = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(P)]
    infos = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(P)]
    steps = [D.getrf_dist_steps(locs[r], descs[r], ipivs[r], infos[r], CudaOps()) for r in range(P)]
    # each generator yields (s, buffer of panel s) at its broadcast point (lookahead
    # order); the 'broadcast' is a device copy from the owner's buffer, then all resume
    items = [next(g) for g in steps]
    for s in range(descs[0].nblocks):
        assert all(it[0] == s for it in items)
        for r in range(P):
            if r != s % P:
                items[r][1].copy_(items[s % P][1])
        items = [next(g, None) for g in steps]
    assert all(it is None for it in items)
    full_out = descs[0].gather([t.cpu() for t in locs]).numpy().view(np.uint32)
    ref, rpiv, rinfo = O.getrf(A)
    assert mismatch(full_out, ref) == 0
    for r in range(P):
        assert np.array_equal(ipivs[r].cpu().numpy(), rpiv) and int(infos[r].cpu()[0]) == rinfo


def test_potrf_dist_p1_cuda(cuda_ok):
    from paper_2401_14117_b200.dist import potrf_dist
    n, nb = 280, 32
    A = O.from_f64_array(SI.config3(n))
    desc = BlockCyclic1D(n, nb, 1, 0)
    loc = desc.scatter(to_dev(A))
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    potrf_dist(loc, desc, info)
    ref, rinfo = O.potrf_lower(A)
    il = np.tril_indices(n)
    assert int(info.cpu()[0]) == rinfo == 0 and mismatch(to_host(loc)[il], ref[il]) == 0


@pytest.mark.parametrize("P", [2, 4])
def test_potrf_dist_emulated_ranks_cuda(cuda_ok, P):
    import paper_2401_14117_b200.dist as D
    n, nb = 190, 16
    A = O.from_f64_array(SI.config3(n))
    full = to_dev(A)
    descs = [BlockCyclic1D(n, nb, P, r) for r in range(P)]
    locs = [d.scatter(full) for d in descs]
    infos = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(P)]
    steps = [D.potrf_dist_steps(locs[r], descs[r], infos[r], D.CudaCholOps()) for r in range(P)]
    items = [next(g) for g in steps]
    for s in range(descs[0].nblocks):
        assert all(it[0] == s for it in items)
        for r in range(P):
            if r != s % P:
                items[r][1].copy_(items[s % P][1])
        items = [next(g, None) for g in steps]
    assert all(it is None for it in items)
    got = descs[0].gather([t.cpu() for t in locs]).numpy().view(np.uint32)
    ref, rinfo = O.potrf_lower(A)
    il = np.tril_indices(n)
    assert mismatch(got[il], ref[il]) == 0 and all(int(i.cpu()[0]) == rinfo for i in infos)


def test_iamax_key_cuda(cuda_ok):
    import paper_2401_14117_b200 as PB
    rng = np.random.default_rng(9)
    pats = O.from_f64_array(SI.normal_matrix((300, 5), 1.0, 9))
    pats[17, 2] = O.P32_NAR
    pats[40, 2] = pats[41, 2]                     # a tie in |a|
    col = to_dev(pats)[:, 2]
    grow = torch.from_numpy(rng.permutation(1000)[:300].astype(np.int32)).cuda()
    key = torch.zeros(1, dtype=torch.int64, device="cuda")
    for row_min in (0, 400, 900, 2000):
        PB.posit_iamax_key(col, grow, row_min, key)
        x = pats[:, 2].astype(np.int64)
        s = np.where(x >= 2 ** 31, x - 2 ** 32, x)
        a = np.where(s < 0, -s, s)
        a = np.where(s == -(2 ** 31), -(2 ** 31), a)
        g = grow.cpu().numpy().astype(np.int64)
        ok = g >= row_min
        ref = int((((a[ok] + 2 ** 31) << 31) | ((2 ** 31 - 1) - g[ok])).max()) if ok.any() else 0
        assert int(key.item()) == ref


def test_getrf_dist2d_1x1_cuda(cuda_ok):
    import socket
    import torch.distributed as dist
    from paper_2401_14117_b200.dist2d import BlockCyclic2D, Groups, getrf_dist2d
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        n, nb = 150, 16
        A = O.from_f64_array(SI.config4(n))
        desc = BlockCyclic2D(n, nb, 1, 1, 0, 0)
        loc = desc.scatter(to_dev(A))
        ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        getrf_dist2d(loc, desc, ipiv, info, Groups(1, 1))
        ref, rpiv, rinfo = O.getrf(A)
        assert mismatch(to_host(loc), ref) == 0
        assert np.array_equal(ipiv.cpu().numpy(), rpiv) and int(info.cpu()[0]) == rinfo
    finally:
        dist.destroy_process_group()
