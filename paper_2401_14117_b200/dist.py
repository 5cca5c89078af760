"""Multi-GPU Posit(32,2) LU: 1 x P column-block-cyclic layout, NCCL panel broadcast.

BASELINE.json north_star (3): "the trailing update is split by column blocks,
2D block-cyclic, with NCCL broadcast of the factored panel and pivot rows over
NVLink".  SURVEY.md 8(e).  The paper itself drives one accelerator over PCIe
(P:435-436); this layer is B200-first, not a port.

Layout.  The n x n matrix is cut into column blocks of nb; rank r of P owns
the blocks j with j mod P == r, stored side by side (ascending j) in one local
row-major n x (nloc) tensor -- all rows, its own columns.

Per panel step s (columns [s nb, s nb + b)), owner o = s mod P:
  1. owner: unblocked LU of its (n - s nb) x b panel in place (posit_getrf_panel:
     pivot by signed-int compare, swap inside the panel, posit division,
     in-panel update), ipiv in global 1-based rows;
  2. owner packs [panel | ipiv | info] into one int32 buffer; ONE broadcast
     (torch.distributed -> ncclBroadcast over NVLink / NVSwitch);
  3. every rank: laswp of the step's b interchanges on all its other columns,
     U12 = L11^-1 A12 (unit-lower TRSM) and A22 <- A22 - L21 U12 (the hot GEMM)
     on its columns right of the panel.
With lookahead the owner of panel s+1 updates and factors it before the rest
of step s's update, and its broadcast overlaps that update (side stream).
No reductions in the data path.  By the order contract (Q6) every
element still receives its products one at a time in ascending k, so the
factors are bit-identical to the single-GPU posit_getrf and to the textbook
loop for every P.

The arithmetic goes through an ``ops`` object.  The product uses ``CudaOps``
(the C ABI of libposit_b200.so on the current CUDA stream); the CPU tests pass
their own implementation of the same five calls to exercise this schedule on
``gloo`` without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class BlockCyclic1D:
    """Column-block-cyclic descriptor: n x n matrix, blocks of nb columns over P ranks."""
    n: int
    nb: int
    nprocs: int
    rank: int

    @property
    def nblocks(self) -> int:
        return (self.n + self.nb - 1) // self.nb

    def owner(self, j: int) -> int:
        return j % self.nprocs

    def block_width(self, j: int) -> int:
        return min(self.nb, self.n - j * self.nb)

    def local_blocks(self, rank: int | None = None) -> list[int]:
        r = self.rank if rank is None else rank
        return list(range(r, self.nblocks, self.nprocs))

    def local_cols(self, rank: int | None = None) -> int:
        return sum(self.block_width(j) for j in self.local_blocks(rank))

    def local_offset(self, j: int) -> int:
        """Column offset of global block j inside its owner's local storage."""
        return sum(self.block_width(i) for i in range(self.owner(j), j, self.nprocs))

    def first_local_after(self, s: int, rank: int | None = None) -> int:
        """Local column offset of this rank's first block with global index > s
        (== local_cols() if none)."""
        off = 0
        for j in self.local_blocks(rank):
            if j > s:
                return off
            off += self.block_width(j)
        return off

    def scatter(self, A: torch.Tensor, rank: int | None = None) -> torch.Tensor:
        """This rank's local columns of the full matrix A (a copy)."""
        cols = [A[:, j * self.nb: j * self.nb + self.block_width(j)] for j in self.local_blocks(rank)]
        if not cols:
            return A.new_empty((self.n, 0))
        return torch.cat(cols, dim=1).contiguous()

    def gather(self, locals_by_rank: list[torch.Tensor]) -> torch.Tensor:
        """Reassemble the full matrix from every rank's local tensor."""
        out = locals_by_rank[0].new_empty((self.n, self.n))
        for r, L in enumerate(locals_by_rank):
            off = 0
            for j in self.local_blocks(r):
                w = self.block_width(j)
                out[:, j * self.nb: j * self.nb + w] = L[:, off: off + w]
                off += w
        return out


def _collective(P: int, group) -> bool:
    """Broadcast whenever a process group exists -- also at P = 1 (bench.py
    --force-dist), so the NCCL / side-stream / record_stream path of the
    schedule runs on a one-GPU lease exactly as it does at P > 1."""
    return P > 1 or group is not None or (dist.is_available() and dist.is_initialized())


class CudaOps:
    """The product arithmetic: libposit_b200.so through the package binding."""

    def __init__(self):
        import paper_2401_14117_b200 as PB
        self.PB = PB

    def getrf_panel(self, P, ipiv, info, row_base):
        self.PB.posit_getrf_panel(P, ipiv, info, row_base=row_base)

    def laswp(self, A, k1, k2, ipiv):
        if A.shape[1] > 0:
            self.PB.posit_laswp(A, k1, k2, ipiv, ipiv_base=0)

    def trsm_llnu(self, L, B):
        if B.shape[1] > 0:
            self.PB.posit_trsm("L", "L", "N", "U", L, B)

    def gemm_minus(self, A, B, C):
        if C.shape[0] > 0 and C.shape[1] > 0:
            self.PB.posit_gemm(A, B, C)


def getrf_dist(A_local: torch.Tensor, desc: BlockCyclic1D, ipiv: torch.Tensor, info: torch.Tensor,
               ops=None, group=None, lookahead: bool = True) -> None:
    """In-place distributed LU with partial pivoting of the n x n matrix whose
    local columns (desc.scatter) are A_local (int32 pattern storage, row-major).

    ipiv (int32, n) receives the global 1-based pivots on EVERY rank; info
    (int32, 1) the first zero-pivot column (1-based) or 0, on every rank.

    Lookahead (CUDA tensors): the owner of panel s+1 updates that panel's
    columns first, factors it and starts its broadcast on a high-priority side
    stream, while every rank's trailing update of step s continues on the
    current stream; the broadcast is awaited only when step s+1 is applied.
    """
    ops = CudaOps() if ops is None else ops
    cuda = A_local.is_cuda and lookahead
    P = desc.nprocs
    if not cuda:
        steps = getrf_dist_steps(A_local, desc, ipiv, info, ops)
        for s, buf in steps:
            if _collective(P, group):
                dist.broadcast(buf, src=desc.owner(s), group=group)
        return
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream(device=A_local.device, priority=-1)
    pending = {}

    class _OnSide:
        def __enter__(self):
            side.wait_stream(main)
            self._ctx = torch.cuda.stream(side)
            self._ctx.__enter__()

        def __exit__(self, *a):
            return self._ctx.__exit__(*a)

    def on_use(s):
        main.wait_stream(side)
        w = pending.pop(s, None)
        if w is not None:
            w.wait()

    steps = getrf_dist_steps(A_local, desc, ipiv, info, ops, panel_ctx=_OnSide, on_use=on_use)
    for s, buf in steps:
        buf.record_stream(side)              # allocated on the main stream, used on the side stream too
        if _collective(P, group):
            with torch.cuda.stream(side):
                side.wait_stream(main)
                pending[s] = dist.broadcast(buf, src=desc.owner(s), group=group, async_op=True)
    main.wait_stream(side)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def getrf_dist_steps(A_local, desc: BlockCyclic1D, ipiv, info, ops, panel_ctx=None, on_use=None):
    """The per-rank schedule of getrf_dist as a generator, in lookahead order.

    It yields (s, buf) once per panel s: buf is the packed
    [panel | ipiv | info] buffer of panel s, filled on the owner; the caller
    broadcasts it (possibly asynchronously).  on_use(s) is called right before
    buf is first read on this rank.  panel_ctx() wraps the owner's work on the
    next panel (its factorisation and packing), e.g. to run it on a side stream.
    Step s: apply panel s (laswp, U12 TRSM); the owner of panel s+1 updates its
    columns of that block, factors and packs it -> yield; then every rank
    updates its remaining trailing columns with step s."""
    panel_ctx = panel_ctx or _Null
    on_use = on_use or (lambda s: None)
    n, nb, me = desc.n, desc.nb, desc.rank
    if A_local.shape != (n, desc.local_cols()):
        raise ValueError(f"A_local has shape {tuple(A_local.shape)}, expected {(n, desc.local_cols())}")
    dev = A_local.device
    info.zero_()
    my_info = torch.zeros(1, dtype=torch.int32, device=dev)
    nloc = A_local.shape[1]
    nblk = desc.nblocks

    def new_buf(s):
        m = n - s * nb
        b = desc.block_width(s)
        return torch.empty(m * b + b + 1, dtype=torch.int32, device=dev)

    def factor_and_pack(s, buf):
        r0, b = s * nb, desc.block_width(s)
        m = n - r0
        lc = desc.local_offset(s)
        Ap = A_local[r0:, lc: lc + b]
        ops.getrf_panel(Ap, ipiv[r0: r0 + b], my_info, r0)
        buf[: m * b].view(m, b).copy_(Ap)
        buf[m * b: m * b + b].copy_(ipiv[r0: r0 + b])
        buf[m * b + b: m * b + b + 1].copy_(my_info)

    buf = new_buf(0)
    if me == desc.owner(0):
        with panel_ctx():
            factor_and_pack(0, buf)
    yield 0, buf
    for s in range(nblk):
        r0, b = s * nb, desc.block_width(s)
        m = n - r0
        o = desc.owner(s)
        on_use(s)
        panel = buf[: m * b].view(m, b)
        if me != o:
            ipiv[r0: r0 + b].copy_(buf[m * b: m * b + b])
        # first zero pivot so far, identical on every rank (the owner's counter is cumulative)
        step_info = buf[m * b + b: m * b + b + 1]
        info.copy_(torch.where(info != 0, info, step_info))
        # interchanges on every local column outside this panel
        if me == o:
            lc = desc.local_offset(s)
            ops.laswp(A_local[:, :lc], r0, r0 + b, ipiv)
            ops.laswp(A_local[:, lc + b:], r0, r0 + b, ipiv)
        else:
            ops.laswp(A_local, r0, r0 + b, ipiv)
        # U12 on the columns right of the panel
        t0 = desc.first_local_after(s)
        if t0 < nloc:
            ops.trsm_llnu(panel[:b], A_local[r0: r0 + b, t0:])
        L21 = panel[b:]
        r1 = r0 + b
        if s + 1 < nblk:
            o1 = desc.owner(s + 1)
            nxt = new_buf(s + 1)
            if me == o1:
                # the next panel's columns first, then factor it (side stream under lookahead)
                lc1 = desc.local_offset(s + 1)
                b1 = desc.block_width(s + 1)
                if r1 < n:
                    ops.gemm_minus(L21, A_local[r0: r1, lc1: lc1 + b1], A_local[r1:, lc1: lc1 + b1])
                with panel_ctx():
                    factor_and_pack(s + 1, nxt)
            yield s + 1, nxt
            # the rest of step s's trailing update
            if t0 < nloc and r1 < n:
                if me == o1:
                    lc1 = desc.local_offset(s + 1)
                    b1 = desc.block_width(s + 1)
                    if t0 < lc1:
                        ops.gemm_minus(L21, A_local[r0: r1, t0: lc1], A_local[r1:, t0: lc1])
                    if lc1 + b1 < nloc:
                        ops.gemm_minus(L21, A_local[r0: r1, lc1 + b1:], A_local[r1:, lc1 + b1:])
                else:
                    ops.gemm_minus(L21, A_local[r0: r1, t0:], A_local[r1:, t0:])
            buf = nxt
        elif t0 < nloc and r1 < n:
            ops.gemm_minus(L21, A_local[r0: r1, t0:], A_local[r1:, t0:])


# ---------------------------------------------------------------- Cholesky ----
# the same 1 x P column-block-cyclic layout for the lower
# Cholesky factorisation.  Per step s the owner factors the diagonal block
# (potf2) and solves the rows below it (L21 = A21 L11^-T), packs the panel and
# its info flag, and broadcasts; every rank then applies the symmetric update
# to its own later column blocks: for block j > s, rows >= j nb,
#     A[r, c] <- A[r, c] (-) L[r, s-block] . L[c, s-block]^T   (c <= r),
# as a SYRK on the diagonal block and an NT GEMM below it.  Same lookahead as
# the LU.  No pivoting, no reductions; bits identical for every P (Q6).

class CudaCholOps:
    """The Cholesky arithmetic through the C ABI (current CUDA stream)."""

    def __init__(self):
        import paper_2401_14117_b200 as PB
        self.PB = PB

    def potrf_block(self, D, info, row_base):
        """Factor the b x b diagonal block D (lower); a failure sets info = row_base + k + 1."""
        loc = torch.zeros(1, dtype=torch.int32, device=D.device)
        self.PB.posit_potrf(D, loc, nb=max(D.shape[0], 1))
        info.copy_(torch.where((info == 0) & (loc != 0), loc + row_base, info))

    def trsm_rltn(self, L, B):
        if B.shape[0] > 0:
            self.PB.posit_trsm("R", "L", "T", "N", L, B)

    def syrk_minus(self, A, C):
        if C.shape[0] > 0:
            self.PB.posit_syrk(A, C)

    def gemm_nt_minus(self, A, B, C):
        if C.shape[0] > 0 and C.shape[1] > 0:
            self.PB.posit_gemm(A, B, C, transb="T")


def potrf_dist(A_local: torch.Tensor, desc: BlockCyclic1D, info: torch.Tensor, ops=None, group=None,
               lookahead: bool = True) -> None:
    """In-place distributed lower Cholesky of the n x n SPD matrix whose local
    column blocks (desc.scatter) are A_local.  info (int32, 1) receives the
    first failing column (1-based) or 0 on every rank; after a failure only
    info and the blocks before the failing one are defined (as posit_potrf)."""
    ops = CudaCholOps() if ops is None else ops
    cuda = A_local.is_cuda and lookahead
    P = desc.nprocs
    if not cuda:
        for s, buf in potrf_dist_steps(A_local, desc, info, ops):
            if _collective(P, group):
                dist.broadcast(buf, src=desc.owner(s), group=group)
        return
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream(device=A_local.device, priority=-1)
    pending = {}

    class _OnSide:
        def __enter__(self):
            side.wait_stream(main)
            self._ctx = torch.cuda.stream(side)
            self._ctx.__enter__()

        def __exit__(self, *a):
            return self._ctx.__exit__(*a)

    def on_use(s):
        main.wait_stream(side)
        w = pending.pop(s, None)
        if w is not None:
            w.wait()

    for s, buf in potrf_dist_steps(A_local, desc, info, ops, panel_ctx=_OnSide, on_use=on_use):
        buf.record_stream(side)
        if _collective(P, group):
            with torch.cuda.stream(side):
                side.wait_stream(main)
                pending[s] = dist.broadcast(buf, src=desc.owner(s), group=group, async_op=True)
    main.wait_stream(side)


def potrf_dist_steps(A_local, desc: BlockCyclic1D, info, ops, panel_ctx=None, on_use=None):
    """The per-rank Cholesky schedule as a generator (lookahead order); yields
    (s, buf) with buf = [panel (n - s nb) x b | info] filled on the owner."""
    panel_ctx = panel_ctx or _Null
    on_use = on_use or (lambda s: None)
    n, nb, me = desc.n, desc.nb, desc.rank
    if A_local.shape != (n, desc.local_cols()):
        raise ValueError(f"A_local has shape {tuple(A_local.shape)}, expected {(n, desc.local_cols())}")
    dev = A_local.device
    info.zero_()
    my_info = torch.zeros(1, dtype=torch.int32, device=dev)
    nblk = desc.nblocks

    def new_buf(s):
        m = n - s * nb
        b = desc.block_width(s)
        return torch.empty(m * b + 1, dtype=torch.int32, device=dev)

    def factor_and_pack(s, buf):
        r0, b = s * nb, desc.block_width(s)
        m = n - r0
        lc = desc.local_offset(s)
        D = A_local[r0: r0 + b, lc: lc + b]
        ops.potrf_block(D, my_info, r0)
        ops.trsm_rltn(D, A_local[r0 + b:, lc: lc + b])
        buf[: m * b].view(m, b).copy_(A_local[r0:, lc: lc + b])
        buf[m * b: m * b + 1].copy_(my_info)

    def update_block(s, panel, j):
        """Block j (> s) of this rank: rows >= j nb get the step-s update."""
        r0, rj, bj = s * nb, j * nb, desc.block_width(j)
        lcj = desc.local_offset(j)
        Lrows = panel[rj - r0:]                        # L[r, s-block] for r >= j nb
        Lj = panel[rj - r0: rj - r0 + bj]              # L[c, s-block] for c in block j
        ops.syrk_minus(Lj, A_local[rj: rj + bj, lcj: lcj + bj])
        if rj + bj < n:
            ops.gemm_nt_minus(Lrows[bj:], Lj, A_local[rj + bj:, lcj: lcj + bj])

    buf = new_buf(0)
    if me == desc.owner(0):
        with panel_ctx():
            factor_and_pack(0, buf)
    yield 0, buf
    for s in range(nblk):
        r0, b = s * nb, desc.block_width(s)
        m = n - r0
        on_use(s)
        panel = buf[: m * b].view(m, b)
        step_info = buf[m * b: m * b + 1]
        info.copy_(torch.where(info != 0, info, step_info))
        mine = [j for j in desc.local_blocks() if j > s]
        if s + 1 < nblk:
            o1 = desc.owner(s + 1)
            nxt = new_buf(s + 1)
            if me == o1:
                update_block(s, panel, s + 1)
                with panel_ctx():
                    factor_and_pack(s + 1, nxt)
            yield s + 1, nxt
            for j in mine:
                if j != s + 1:
                    update_block(s, panel, j)
            buf = nxt


# ------------------------------------------------------------------ GEMM ------
# SURVEY 8(e) "GEMM (C2): split C by column blocks.  Each rank needs A
# (broadcast) and its B slab.  No split-K (forbidden by c4) and no reduction."
# One m x n x k problem over P ranks (strong scaling): rank r owns the
# contiguous column slab [c0_r, c1_r) of B and C; A lives on rank `src` and is
# sent to every rank with ONE broadcast per call; then each rank runs
# C_r <- C_r - A . B_r on its own slab.  Every output element's chain is the
# single-GPU one (Q6), so the gathered C is bit-identical for every P.

def col_slab(n: int, nprocs: int, rank: int) -> tuple[int, int]:
    """[c0, c1) of rank's column slab: contiguous, balanced, multiples of 4
    columns (16-byte rows for the kernels' quad loads) except the last."""
    q = (n + 4 * nprocs - 1) // (4 * nprocs) * 4
    c0 = min(n, rank * q)
    return c0, min(n, c0 + q)


def gemm_colsplit(A: torch.Tensor, B_local: torch.Tensor, C_local: torch.Tensor, src: int = 0,
                  ops=None, group=None) -> None:
    """C_local <- C_local - A . B_local on this rank's column slab, after ONE
    broadcast of A (m x k, allocated on every rank; its contents matter on
    `src` only) from rank `src`."""
    ops = CudaOps() if ops is None else ops
    if dist.is_available() and dist.is_initialized():
        dist.broadcast(A, src=src, group=group)
    ops.gemm_minus(A, B_local, C_local)
