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
