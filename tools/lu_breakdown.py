"""Where the LU time goes: posit_getrf at configs[4] s = 0 (n = 8192, nb = 256;
LB_N = 16384 for configs[3]) next to the same step sequence's pieces timed
standalone back to back on one stream — the trailing GEMMs (r x r, K = 256,
r = n - 256 (s + 1)), the panels ((r + 256) x 256, partial pivoting), the
row-panel TRSMs (256 x r) — so the lookahead's overlap and each piece's own
rate can be read off (the companion of tools/chol_breakdown.py).

    python tools/lu_breakdown.py          # one JSON line
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

n, nb = int(os.environ.get("LB_N", "8192")), 256
dev = "cuda"
A0 = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(n, SI.C5_SEED)).to(dev))
ipiv = torch.zeros(n, dtype=torch.int32, device=dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def full():
    A = A0.clone()
    PB.posit_getrf(A, ipiv, info, nb=nb)


W = A0.clone()
steps = range(n // nb - 1)


def gemms():
    for s in steps:
        r0 = (s + 1) * nb
        # fixed operands (the first block column / row): values stay in the fast-path range
        PB.posit_gemm(A0[r0:, :nb], A0[:nb, r0:], W[r0:, r0:])


Pn = A0[:, :nb].clone()
PB.posit_getrf_panel(Pn, ipiv[:nb], info, 0)
L11 = Pn[:nb].clone()


def panels():
    for s in range(n // nb):
        P = A0[s * nb:, :nb].clone()
        PB.posit_getrf_panel(P, ipiv[:nb], info, 0)


def panel_copies():
    for s in range(n // nb):
        A0[s * nb:, :nb].clone()


Bs = [A0[:nb, (s + 1) * nb:].clone() for s in steps]   # fresh right-hand sides: no repeated solves


def trsms():
    for s in steps:
        PB.posit_trsm("L", "L", "N", "U", L11, Bs[s])


t_copy = timed(lambda: A0.clone())
t_full = timed(full) - t_copy
t_gemm = timed(gemms)
t_panel = timed(panels) - timed(panel_copies)
t_trsm = timed(trsms)
flops = 2 * n ** 3 / 3
gemm_flops = sum(2 * (n - (s + 1) * nb) ** 2 * nb for s in steps)
print(json.dumps({"n": n, "nb": nb, "getrf_ms": t_full, "getrf_gflops": flops / t_full / 1e6,
                  "gemm_sum_ms": t_gemm, "gemm_gflops": gemm_flops / t_gemm / 1e6,
                  "panel_sum_ms": t_panel, "trsm_sum_ms": t_trsm,
                  "serial_sum_ms": t_gemm + t_panel + t_trsm,
                  "note": "pieces standalone back to back; getrf overlaps them (lookahead); laswp not included"}))
