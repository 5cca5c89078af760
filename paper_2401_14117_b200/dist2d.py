"""Multi-GPU Posit(32,2) LU on a 2D Pr x Pc block-cyclic process grid.

BASELINE.json north_star (3), "2D block-cyclic"; the
Pr > 1 grids.  (dist.py is the Pr = 1 case with lookahead, the default.)

Layout: nb x nb block (I, J) lives on process (I mod Pr, J mod Pc); a rank
stores its block rows x block columns side by side (ascending global index) as
one row-major tensor.  Rank = pr * Pc + pc.

Per panel step s (column block s on process column pcs = s mod Pc):
  1. panel, column by column, by the Pr ranks of process column pcs: local
     pivot key (posit_iamax_key: larger |a| by signed-int compare, ties ->
     smaller global row, Q10) -> MAX all-reduce over the process column ->
     the rows g and p of the panel shared by a sum all-reduce (zeros
     elsewhere) -> swap,
     one posit division per multiplier (Q8, Q11 for a zero pivot), rank-1
     update of the panel's later columns (posit_gemm with K = 1);
  2. ipiv/info to every rank; the factored panel along each process row;
  3. the step's row interchanges on every other column: the touched rows are
     summed (exact: zeros elsewhere) over the process column, then permuted;
  4. U12 = L11^-1 A12 on process row s mod Pr, broadcast down each process
     column; 5. A22 -= L21 U12 on every rank's own rows and columns.
Every element still receives its products one at a time in ascending k, so the
factors are bit-identical to the 1-GPU posit_getrf and the textbook loop for
every grid (Q6).  The column-by-column panel costs one all-reduce
and two broadcasts per column (SURVEY 8(e) expects this to be slower than
Pr = 1 at n = 16384); it exists for grids where a column block does not fit.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

KEY_ROW_MASK = (1 << 31) - 1


@dataclass(frozen=True)
class BlockCyclic2D:
    n: int
    nb: int
    Pr: int
    Pc: int
    pr: int
    pc: int

    @property
    def nblocks(self) -> int:
        return (self.n + self.nb - 1) // self.nb

    def _idx(self, p, P):
        out = []
        for I in range(p, self.nblocks, P):
            out.extend(range(I * self.nb, min((I + 1) * self.nb, self.n)))
        return np.array(out, dtype=np.int64)

    def rows(self, pr=None):
        return self._idx(self.pr if pr is None else pr, self.Pr)

    def cols(self, pc=None):
        return self._idx(self.pc if pc is None else pc, self.Pc)

    def owner_row(self, g):
        return (g // self.nb) % self.Pr

    def owner_col(self, g):
        return (g // self.nb) % self.Pc

    def local_row(self, g):
        """Local index of global row g on its owner."""
        return ((g // self.nb) // self.Pr) * self.nb + g % self.nb

    def local_col(self, g):
        return ((g // self.nb) // self.Pc) * self.nb + g % self.nb

    def first_local_row_at_least(self, g, pr=None):
        r = self.rows(pr)
        return int(np.searchsorted(r, g))

    def first_local_col_at_least(self, g, pc=None):
        c = self.cols(pc)
        return int(np.searchsorted(c, g))

    def scatter(self, A: torch.Tensor) -> torch.Tensor:
        r = torch.from_numpy(self.rows()).to(A.device)
        c = torch.from_numpy(self.cols()).to(A.device)
        return A.index_select(0, r).index_select(1, c).contiguous()

    def gather(self, locals_by_rank) -> torch.Tensor:
        out = locals_by_rank[0].new_empty((self.n, self.n))
        for rank, L in enumerate(locals_by_rank):
            pr, pc = divmod(rank, self.Pc)
            r = torch.from_numpy(self.rows(pr))
            c = torch.from_numpy(self.cols(pc))
            out[r.unsqueeze(1), c.unsqueeze(0)] = L
        return out


class Groups:
    """Process-row and process-column groups (every rank creates all of them, same order)."""

    def __init__(self, Pr, Pc, backend=None):
        self.col = [dist.new_group([pr * Pc + pc for pr in range(Pr)], backend=backend) for pc in range(Pc)]
        self.row = [dist.new_group([pr * Pc + pc for pc in range(Pc)], backend=backend) for pr in range(Pr)]


class CudaOps2D:
    """The arithmetic through the C ABI (current CUDA stream)."""

    def __init__(self):
        import paper_2401_14117_b200 as PB
        self.PB = PB

    def iamax_key(self, col, grow, row_min, key):
        self.PB.posit_iamax_key(col, grow, row_min, key)

    def div_rows(self, col, v):
        """col (strided column view) <- col (/) v, elementwise."""
        if col.shape[0] == 0:
            return
        c = col.contiguous()
        d = torch.full_like(c, int(v) - (1 << 32) if v >= (1 << 31) else int(v))
        col.copy_(self.PB.posit_vec_op("div", c, d))

    def rank1_minus(self, l, u, C):
        if C.shape[0] > 0 and C.shape[1] > 0:
            self.PB.posit_gemm(l, u, C)

    def trsm_llnu(self, L, B):
        if B.shape[0] > 0 and B.shape[1] > 0:
            self.PB.posit_trsm("L", "L", "N", "U", L, B)

    def gemm_minus(self, A, B, C):
        if C.shape[0] > 0 and C.shape[1] > 0 and A.shape[1] > 0:
            self.PB.posit_gemm(A, B, C)


def _u32(x):
    return int(x) & 0xFFFFFFFF


def getrf_dist2d(A_local, desc: BlockCyclic2D, ipiv, info, groups: Groups, ops=None):
    """In-place LU with partial pivoting of the n x n matrix whose local part
    (desc.scatter) is A_local, on the Pr x Pc grid.  ipiv (int32, n) and info
    (int32, 1) are filled identically on every rank."""
    ops = CudaOps2D() if ops is None else ops
    n, nb, Pr, Pc, me_r, me_c = desc.n, desc.nb, desc.Pr, desc.Pc, desc.pr, desc.pc
    dev = A_local.device
    colg, rowg = groups.col[me_c], groups.row[me_r]
    grow = torch.from_numpy(desc.rows().astype(np.int32)).to(dev)
    info.zero_()
    ipiv.zero_()
    nloc_c = A_local.shape[1]
    for s in range(desc.nblocks):
        r0, b = s * nb, min(nb, n - s * nb)
        pcs, prs = s % Pc, s % Pr
        lc0 = desc.local_col(r0) if me_c == pcs else -1
        piv_buf = torch.zeros(b + 1, dtype=torch.int32, device=dev)
        # ---- 1. the panel (process column pcs) ---------------------------------
        if me_c == pcs:
            P = A_local[:, lc0: lc0 + b]
            key = torch.zeros(1, dtype=torch.int64, device=dev)
            for jj in range(b):
                g = r0 + jj
                ops.iamax_key(P[:, jj], grow, g, key)
                if Pr > 1:
                    dist.all_reduce(key, op=dist.ReduceOp.MAX, group=colg)
                p = KEY_ROW_MASK - (int(key.item()) & KEY_ROW_MASK)
                rows_gp = torch.zeros(2, b, dtype=torch.int32, device=dev)
                if desc.owner_row(g) == me_r:
                    rows_gp[0].copy_(P[desc.local_row(g)])
                if desc.owner_row(p) == me_r:
                    rows_gp[1].copy_(P[desc.local_row(p)])
                if Pr > 1:
                    dist.all_reduce(rows_gp, op=dist.ReduceOp.SUM, group=colg)   # exact: zeros elsewhere
                v = _u32(rows_gp[1, jj].item())
                piv_buf[jj] = p + 1
                if v != 0 and p != g:
                    if desc.owner_row(g) == me_r:
                        P[desc.local_row(g)].copy_(rows_gp[1])
                    if desc.owner_row(p) == me_r:
                        P[desc.local_row(p)].copy_(rows_gp[0])
                elif v == 0 and int(piv_buf[b]) == 0:
                    piv_buf[b] = g + 1
                pivrow = rows_gp[1] if (v != 0 and p != g) else rows_gp[0]
                lr = desc.first_local_row_at_least(g + 1)
                if v != 0:
                    ops.div_rows(P[lr:, jj], v)
                if jj + 1 < b:
                    ops.rank1_minus(P[lr:, jj: jj + 1], pivrow[jj + 1:].view(1, -1), P[lr:, jj + 1:])
        # ---- 2. ipiv / info everywhere, the panel along each process row ---------
        if Pr * Pc > 1:       # every rank of process column pcs holds the same piv_buf; send rank (prs, pcs)'s
            dist.broadcast(piv_buf, src=prs * Pc + pcs)
        ipiv[r0: r0 + b].copy_(piv_buf[:b])
        if int(info[0]) == 0 and int(piv_buf[b]) != 0:
            info[0] = piv_buf[b]
        Lp = torch.empty(A_local.shape[0], b, dtype=torch.int32, device=dev)
        if me_c == pcs:
            Lp.copy_(A_local[:, lc0: lc0 + b])
        if Pc > 1:
            dist.broadcast(Lp, src=me_r * Pc + pcs, group=rowg)
        # ---- 3. the step's row interchanges on every other local column ----------
        touched = []
        for jj in range(b):
            g, p = r0 + jj, int(piv_buf[jj]) - 1
            for x in (g, p):
                if x not in touched:
                    touched.append(x)
        content = {x: x for x in touched}            # row position -> original row now there
        for jj in range(b):
            g, p = r0 + jj, int(piv_buf[jj]) - 1
            content[g], content[p] = content[p], content[g]
        old = torch.zeros(len(touched), nloc_c, dtype=torch.int32, device=dev)
        for t, x in enumerate(touched):
            if desc.owner_row(x) == me_r:
                old[t].copy_(A_local[desc.local_row(x)])
        if Pr > 1:
            dist.all_reduce(old, op=dist.ReduceOp.SUM, group=colg)
        pos = {x: t for t, x in enumerate(touched)}
        keep = None
        if me_c == pcs:
            keep = torch.ones(nloc_c, dtype=torch.bool, device=dev)
            keep[lc0: lc0 + b] = False
        for x in touched:
            if desc.owner_row(x) == me_r and content[x] != x:
                src = old[pos[content[x]]]
                row = A_local[desc.local_row(x)]
                if keep is None:
                    row.copy_(src)
                else:
                    row[keep] = src[keep]
        # ---- 4. U12 on process row prs, down each process column -------------------
        lct = desc.first_local_col_at_least(r0 + b)
        ntr = nloc_c - lct
        U12 = torch.empty(b, ntr, dtype=torch.int32, device=dev)
        if me_r == prs:
            lr0 = desc.local_row(r0)
            if ntr > 0:
                ops.trsm_llnu(Lp[lr0: lr0 + b], A_local[lr0: lr0 + b, lct:])
            U12.copy_(A_local[lr0: lr0 + b, lct:])
        if Pr > 1 and ntr > 0:
            dist.broadcast(U12, src=prs * Pc + me_c, group=colg)
        # ---- 5. trailing update on this rank's rows and columns --------------------
        lrt = desc.first_local_row_at_least(r0 + b)
        if ntr > 0 and lrt < A_local.shape[0]:
            ops.gemm_minus(Lp[lrt:], U12, A_local[lrt:, lct:])
