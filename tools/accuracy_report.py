"""Accuracy report (separate from parity): the paper's Eq.4 / Eq.5 error study
(Fig cho_err) on the GPU factors, next to binary32 LAPACK.

    python tools/accuracy_report.py [--quick] [--out profiles/accuracy.jsonl]

For each matrix A (binary64): x_sol = 1/sqrt(N), b = A x_sol in
binary64.  Posit: A and b rounded once to Posit(32,2) (posit_from_f64),
posit_getrf/potrf + posit_getrs/potrs on the GPU, x back to binary64 exactly.
binary32: A and b rounded to float32, LAPACK sgetrf/sgetrs or spotrf/spotrs
(scipy); and (n <= 2048) binary32 with the posit path's own algorithm and
operation order (numpy float32 textbook loops, no FMA), so that difference
isolates the number format.  binary64: LAPACK dgesv, for the forward error (reading Q18).
  e_X      = |b - A x_X| / |b|                         (Eq.4, 2-norm, binary64)
  digits   = log10(e_binary32 / e_posit)               (Eq.5; > 0: posit better)
  fwd_X    = -log10(|x_X - x_64| / |x_64|)             (forward-error digits)
Workloads: the BASELINE configs (C1, C3, C4 at n = 4096 unless --full, C5's
2^s sweep) and the paper's sigma sweep (N(0, sigma^2) for LU, A = X^T X for
Cholesky).  Paper context: posit better by ~0.8 digits (LU)
and ~0.5 (Cholesky) at sigma = 1, no advantage at sigma >= 1e2.
"""
import argparse
import json
import os
import sys

import numpy as np
import scipy.linalg as sla
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402


def _err(A, b, x):
    return float(np.linalg.norm(b - A @ x) / np.linalg.norm(b))


def _fwd(x, x64):
    return float(-np.log10(max(np.linalg.norm(x - x64) / np.linalg.norm(x64), 1e-300)))


def _lu32_same_order(A, b):
    """binary32 with the posit path's operation order: textbook
    right-looking kij LU with partial pivoting (ties -> smallest row), one division per
    multiplier, every product and difference rounded to binary32 (numpy float32, no FMA);
    solves in the Q21 order (forward ascending k, back descending k)."""
    A = A.astype(np.float32).copy()
    b = b.astype(np.float32).copy()
    n = A.shape[0]
    piv = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        if p != k:
            A[[k, p]] = A[[p, k]]
            piv[[k, p]] = piv[[p, k]]
        if A[k, k] != 0:
            A[k + 1:, k] = A[k + 1:, k] / A[k, k]
        A[k + 1:, k + 1:] = A[k + 1:, k + 1:] - np.outer(A[k + 1:, k], A[k, k + 1:]).astype(np.float32)
    y = b[piv]
    for k in range(n):                                   # forward, column-oriented (ascending k)
        y[k + 1:] = y[k + 1:] - (A[k + 1:, k] * y[k]).astype(np.float32)
    for k in range(n - 1, -1, -1):                       # back, column-oriented (descending k)
        y[k] = y[k] / A[k, k]
        y[:k] = y[:k] - (A[:k, k] * y[k]).astype(np.float32)
    return y.astype(np.float64)


def _chol32_same_order(A, b):
    A = A.astype(np.float32).copy()
    y = b.astype(np.float32).copy()
    n = A.shape[0]
    for k in range(n):
        if A[k, k] <= 0:
            return np.full(n, np.nan)
        A[k, k] = np.sqrt(A[k, k])
        A[k + 1:, k] = A[k + 1:, k] / A[k, k]
        A[k + 1:, k + 1:] = A[k + 1:, k + 1:] - np.outer(A[k + 1:, k], A[k + 1:, k]).astype(np.float32)
    for k in range(n):
        y[k] = y[k] / A[k, k]
        y[k + 1:] = y[k + 1:] - (A[k + 1:, k] * y[k]).astype(np.float32)
    for k in range(n - 1, -1, -1):
        y[k] = y[k] / A[k, k]
        y[:k] = y[:k] - (A[k, :k] * y[k]).astype(np.float32)
    return y.astype(np.float64)


def study(name, A, kind, nb=256, same_order_max=2048):
    n = A.shape[0]
    x_sol = np.full(n, 1.0 / np.sqrt(n))
    b = A @ x_sol
    dA = PB.posit_from_f64(torch.from_numpy(A).cuda())
    db = PB.posit_from_f64(torch.from_numpy(b).cuda())
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    if kind == "lu":
        ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
        PB.posit_getrf(dA, ipiv, info, nb=nb)
        PB.posit_getrs(dA, ipiv, db)
        f32 = sla.lu_factor(A.astype(np.float32), check_finite=False)
        x32 = sla.lu_solve(f32, b.astype(np.float32), check_finite=False)
    else:
        PB.posit_potrf(dA, info, nb=nb)
        PB.posit_potrs(dA, db)
        try:
            c32 = sla.cho_factor(A.astype(np.float32), lower=True, check_finite=False)
            x32 = sla.cho_solve(c32, b.astype(np.float32), check_finite=False)
        except np.linalg.LinAlgError:           # spotrf: not positive definite in binary32
            x32 = np.full(n, np.nan, np.float32)
    xp = PB.posit_to_f64(db).cpu().numpy()
    x64 = np.linalg.solve(A, b)
    ep, e32 = _err(A, b, xp), _err(A, b, x32.astype(np.float64))
    ok = ep > 0 and np.isfinite(ep) and np.isfinite(e32)
    r = {"case": name, "kind": kind, "n": n, "info": int(info.cpu()[0]), "e_posit": ep, "e_binary32": e32,
         "digits_eq5": float(np.log10(e32 / ep)) if ok else None,
         "fwd_digits_posit": _fwd(xp, x64), "fwd_digits_binary32": _fwd(x32.astype(np.float64), x64)}
    if n <= same_order_max:
        # the same algorithm and operation order in binary32: isolates the number format
        xs = _lu32_same_order(A, b) if kind == "lu" else _chol32_same_order(A, b)
        es = _err(A, b, xs)
        r["e_binary32_same_order"] = es
        r["digits_vs_same_order"] = float(np.log10(es / ep)) if (ep > 0 and np.isfinite(es)) else None
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "accuracy.jsonl"))
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "w")

    def emit(r):
        print(json.dumps(r), flush=True)
        out.write(json.dumps(r) + "\n")
        out.flush()

    emit(study("C1 LU n=256 U[-1,1) seed 0", SI.config1(), "lu", nb=32))
    n4 = 16384 if args.full else 4096
    emit(study(f"C4 recipe LU n={n4} U[-1,1) seed 3", SI.config4(n4), "lu"))
    n3 = 8192 if not args.quick else 2048
    emit(study(f"C3 recipe Cholesky n={n3} GG^T/n+I seed 2", SI.config3(n3), "chol"))
    n5 = 8192 if not args.quick else 2048
    for s in SI.C5_SHIFTS:
        emit(study(f"C5 recipe LU n={n5} U[-1,1)*2^{s} seed 4", SI.config5(s, n5), "lu"))
    # the paper's sigma sweep (Fig cho_err): N(0, sigma^2) for LU, A = X^T X for Cholesky
    for N in ((512, 1024) if args.quick else (512, 1024, 2048, 4096)):
        for sigma in (1e-2, 1.0, 1e2, 1e4, 1e6):
            X = SI.normal_matrix((N, N), sigma, 100 + N)
            emit(study(f"sigma sweep LU N={N} sigma={sigma:g}", X, "lu"))
            emit(study(f"sigma sweep Cholesky N={N} sigma={sigma:g} (A = X^T X)", X.T @ X, "chol"))
    out.close()


if __name__ == "__main__":
    main()
