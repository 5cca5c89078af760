"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): GEMM NN/NT/SYRK, LU (recursive panel, cooperative leaf,
lookahead), Cholesky (potf2 leaf, fused TRSM, lookahead), TRSMs, laswp,
getrs/potrs, conversions.  Exits 0 if every result matches the oracle.

    compute-sanitizer --tool racecheck python tests/sanitize_small.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402
from oracle import oracle as O  # noqa: E402


def dev(p):
    return torch.from_numpy(np.ascontiguousarray(p, np.uint32).view(np.int32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def main():
    bad = 0
    A, B, C = (O.from_f64_array(x) for x in SI.config2(n=150, m=70, k=40))
    dC = dev(C)
    PB.posit_gemm(dev(A), dev(B), dC)
    bad += int(np.count_nonzero(host(dC) != O.gemm(A, B, C)))
    S = O.from_f64_array(SI.normal_matrix((90, 90), 1.0, 3))
    X = O.from_f64_array(SI.normal_matrix((90, 40), 1.0, 4))
    dS = dev(S)
    PB.posit_syrk(dev(X), dS)
    il = np.tril_indices(90)
    bad += int(np.count_nonzero(host(dS)[il] != O.syrk_lower(X, S)[il]))
    L = O.from_f64_array(SI.config4(300))
    dL = dev(L)
    ipiv = torch.zeros(300, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    PB.posit_getrf(dL, ipiv, info, nb=64)
    ref, rpiv, _ = O.getrf(L)
    bad += int(np.count_nonzero(host(dL) != ref)) + int(not np.array_equal(ipiv.cpu().numpy(), rpiv))
    b = O.from_f64_array(SI.normal_matrix((300,), 1.0, 5))
    db = dev(b)
    PB.posit_getrs(dL, ipiv, db)
    bad += int(np.count_nonzero(host(db) != O.getrs(ref, rpiv, b)))
    H = O.from_f64_array(SI.config3(260))
    dH = dev(H)
    PB.posit_potrf(dH, info, nb=64)
    refh, _ = O.potrf_lower(H)
    il = np.tril_indices(260)
    bad += int(np.count_nonzero(host(dH)[il] != refh[il]))
    bb = O.from_f64_array(SI.normal_matrix((260,), 1.0, 6))
    db = dev(bb)
    PB.posit_potrs(dH, db)
    bad += int(np.count_nonzero(host(db) != O.potrs_lower(refh, bb)))
    print("mismatches", bad)
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
