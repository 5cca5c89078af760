"""Time posit_getrf / posit_potrf on the BASELINE configs and break one LU
panel step into its parts (run under gpurun; CUDA events on the current stream).

    python tools/time_lapack.py [--quick]
Prints one JSON object per line.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402


def ev_stats(fn, reps):
    """median and best of `reps` timed runs (CUDA events), SURVEY 8(d) timing protocol."""
    ts = [ev_time(fn)[0] for _ in range(reps)]
    return float(np.median(ts)), float(min(ts))


def ev_time(fn, reps=1, warm=False):
    if warm:
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


def dev_pats(x):
    return PB.posit_from_f64(torch.from_numpy(x).cuda())


def lu(name, A64, nb, reps=1):
    n = A64.shape[0]
    A0 = dev_pats(A64)
    A = A0.clone()
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")

    def run():
        A.copy_(A0)
        PB.posit_getrf(A, ipiv, info, nb=nb)
    run()
    ms, best = ev_stats(run, reps)
    print(json.dumps({"case": name, "n": n, "nb": nb, "reps": reps, "ms": ms, "best_ms": best,
                      "gflops": 2 * n ** 3 / 3 / ms / 1e6, "best_gflops": 2 * n ** 3 / 3 / best / 1e6,
                      "info": int(info.cpu()[0])}), flush=True)


def chol(name, A64, nb, reps=1):
    n = A64.shape[0]
    A0 = dev_pats(A64)
    A = A0.clone()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")

    def run():
        A.copy_(A0)
        PB.posit_potrf(A, info, nb=nb)
    run()
    ms, best = ev_stats(run, reps)
    print(json.dumps({"case": name, "n": n, "nb": nb, "reps": reps, "ms": ms, "best_ms": best,
                      "gflops": n ** 3 / 3 / ms / 1e6, "best_gflops": n ** 3 / 3 / best / 1e6,
                      "info": int(info.cpu()[0])}), flush=True)


def lu_step_breakdown(n, nb, s):
    """Parts of LU panel step s on an n x n U[-1,1) matrix (state: unfactored, shapes as in step s)."""
    A = dev_pats(SI.lu_matrix(n, 3))
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    r0 = s * nb
    m = n - r0
    P = A[r0:, r0:r0 + nb]
    out = {"case": "lu_step", "n": n, "nb": nb, "step": s}
    Pc = P.clone()
    out["panel_ms"], out["panel_host_ms"] = ev_time(lambda: (P.copy_(Pc), PB.posit_getrf_panel(P, ipiv[r0:r0 + nb], info, r0)),
                                                    warm=True)
    out["laswp_ms"], _ = ev_time(lambda: PB.posit_laswp(A[:, r0 + nb:], r0, r0 + nb, ipiv), warm=True)
    B = A[r0:r0 + nb, r0 + nb:]
    Bc = B.clone()
    out["trsm_ms"], out["trsm_host_ms"] = ev_time(lambda: (B.copy_(Bc), PB.posit_trsm("L", "L", "N", "U", P[:nb], B)), warm=True)
    C = A[r0 + nb:, r0 + nb:]
    Cc = C.clone()
    out["gemm_ms"], _ = ev_time(lambda: (C.copy_(Cc), PB.posit_gemm(P[nb:], B, C)))
    out["copy_ms"], _ = ev_time(lambda: C.copy_(Cc))
    out["gemm_gflops"] = 2.0 * (m - nb) * (n - r0 - nb) * nb / (out["gemm_ms"] - out["copy_ms"]) / 1e6
    print(json.dumps(out), flush=True)


def main():
    quick = "--quick" in sys.argv
    # SURVEY 8(d) timing protocol: C1, C3, C5 x 5 (and every C5 shift), C4 x 3; median and best
    lu("C1", SI.config1(), SI.C1_NB, reps=5)
    lu_step_breakdown(16384, 256, 0)
    lu_step_breakdown(16384, 256, 48)
    for sh in ((0,) if quick else SI.C5_SHIFTS):
        lu(f"C5 s={sh}", SI.config5(sh), SI.C5_NB, reps=1 if quick else 5)
    chol("C3", SI.config3(), SI.C3_NB, reps=1 if quick else 5)
    if not quick:
        lu("C4 (1 GPU)", SI.config4(), SI.C4_NB, reps=3)


if __name__ == "__main__":
    main()
