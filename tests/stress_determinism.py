"""Repeat the lookahead LU / Cholesky / GEMM many times and check the output
bits never change (races in the cooperative leaf, the side stream or the
fused kernels would show up as run-to-run differences).

    python tests/stress_determinism.py [reps]
"""
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402


def sha(t):
    torch.cuda.synchronize()
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    bad = 0
    A0 = PB.posit_from_f64(torch.from_numpy(SI.config4(3000)).cuda())
    S0 = PB.posit_from_f64(torch.from_numpy(SI.config3(3000)).cuda())
    G = [PB.posit_from_f64(torch.from_numpy(x).cuda()) for x in SI.config2(n=1500, m=1300, k=700)]
    ipiv = torch.zeros(3000, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    ref = {}
    for r in range(reps):
        A = A0.clone()
        PB.posit_getrf(A, ipiv, info, nb=256)
        S = S0.clone()
        PB.posit_potrf(S, info, nb=256)
        C = G[2].clone()
        PB.posit_gemm(G[0], G[1], C)
        h = {"lu": sha(A) + sha(ipiv), "chol": sha(torch.tril(S)), "gemm": sha(C)}
        if r == 0:
            ref = h
        elif h != ref:
            bad += 1
            print("run", r, "differs", h, ref)
    print("runs", reps, "differing", bad, ref)
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
