"""Subprocess worker of tests/test_gpu_switches.py (test infrastructure).

The library reads its POSIT_* traversal switches once per process, so every
switch setting runs in a fresh process: this script loads the inputs the
parent wrote (numpy uint32 patterns), runs the requested C-ABI calls on the
GPU under the environment it was started with, and writes the outputs back.
It computes nothing itself and never touches the oracle; the parent compares.

    python tests/switch_worker.py <in.npz> <out.npz> <job>

job "gemm":  NN, NT, TN GEMM (C -= op(A) op(B)) and the lower SYRK
             (S -= As As^T) on the parent's operands;
job "lapack": posit_getrf (nb 256) and posit_potrf (nb 256) on the parent's
             matrices.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402


def dev(p):
    return torch.from_numpy(np.ascontiguousarray(p, np.uint32).view(np.int32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32).copy()


def main():
    src, dst, job = sys.argv[1], sys.argv[2], sys.argv[3]
    X = np.load(src)
    out = {}
    if job == "gemm":
        for name, (a, b, ta, tb) in {"nn": ("A", "B", "N", "N"), "nt": ("A", "Bt", "N", "T"),
                                     "tn": ("At", "B", "T", "N")}.items():
            dC = dev(X["C"])
            PB.posit_gemm(dev(X[a]), dev(X[b]), dC, transa=ta, transb=tb)
            out[name] = host(dC)
        dS = dev(X["S"])
        PB.posit_syrk(dev(X["As"]), dS)          # lower triangle of S -= As As^T
        out["syrk"] = host(dS)
    else:
        n = X["L"].shape[0]
        dA = dev(X["L"])
        ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        PB.posit_getrf(dA, ipiv, info, nb=256)
        out["lu"], out["ipiv"], out["lu_info"] = host(dA), ipiv.cpu().numpy(), info.cpu().numpy()
        dS = dev(X["P"])
        PB.posit_potrf(dS, info, nb=256)
        out["chol"], out["chol_info"] = host(dS), info.cpu().numpy()
    np.savez(dst, **out)


if __name__ == "__main__":
    main()
