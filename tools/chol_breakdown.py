"""Where C3's time goes: posit_potrf at configs[2] (n = 8192, nb = 256) next to
the same step sequence's pieces timed standalone back to back on one stream —
the trailing SYRKs (r x r lower, K = 256, r = n - 256 (s + 1)), the TRSMs
(r x 256) and the 256 x 256 diagonal factorisations — so the schedule's
overlap (lookahead) and each piece's own rate can be read off.

    python tools/chol_breakdown.py          # one JSON line
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

n, nb = int(os.environ.get("CB_N", "8192")), 256
dev = "cuda"
A0 = PB.posit_from_f64(torch.from_numpy(SI.config3(n)).to(dev))
info = torch.zeros(1, dtype=torch.int32, device=dev)
D0 = PB.posit_from_f64(torch.from_numpy(SI.config3(nb)).to(dev))


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
    PB.posit_potrf(A, info, nb=nb)


W = A0.clone()
steps = range(n // nb - 1)


def syrks():
    for s in steps:
        r0 = (s + 1) * nb
        PB.posit_syrk(A0[r0:, :nb], W[r0:, r0:])   # fixed operand: values stay in the fast-path range


L11 = PB.posit_from_f64(torch.from_numpy(SI.config3(nb)).to(dev))
PB.posit_potrf(L11, info, nb=nb)
Bt = A0[:, :nb].clone()


def trsms():
    for s in steps:
        r = n - (s + 1) * nb
        PB.posit_trsm("R", "L", "T", "N", L11, Bt[:r])


def potf2s():
    for s in range(n // nb):
        D = D0.clone()
        PB.posit_potrf(D, info, nb=nb)


t_copy = timed(lambda: A0.clone())
t_full = timed(full) - t_copy
t_syrk = timed(syrks)
t_trsm = timed(trsms)
t_potf = timed(potf2s) - (n // nb) * timed(lambda: D0.clone(), reps=5)
flops = n ** 3 / 3
syrk_flops = sum((n - (s + 1) * nb) * (n - (s + 1) * nb + 1) / 2 * nb * 2 for s in steps)
print(json.dumps({"n": n, "nb": nb, "potrf_ms": t_full, "potrf_gflops": flops / t_full / 1e6,
                  "syrk_sum_ms": t_syrk, "syrk_gflops": syrk_flops / t_syrk / 1e6,
                  "trsm_sum_ms": t_trsm, "potf2_sum_ms": t_potf,
                  "serial_sum_ms": t_syrk + t_trsm + t_potf,
                  "note": "pieces standalone back to back; potrf overlaps them (lookahead)"}))
