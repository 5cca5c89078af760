"""One warm-up + one profiled posit_gemm launch (for ncu).

    python tools/prof_gemm.py                       # configs[1]: 4096^3 NN
    PROF_SHAPE=16128,16128,256 python tools/prof_gemm.py   # the first C4 trailing update
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

shape = os.environ.get("PROF_SHAPE")
if shape:
    m, n, k = (int(x) for x in shape.split(","))
    A = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(max(m, k), 3)[:m, :k].copy()).cuda())
    B = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(max(k, n), 4)[:k, :n].copy()).cuda())
    C0 = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(max(m, n), 5)[:m, :n].copy()).cuda())
else:
    m = int(os.environ.get("PROF_M", "4096"))
    A64, B64, C64 = SI.config2(n=m, m=m, k=m)
    A = PB.posit_from_f64(torch.from_numpy(A64).cuda())
    B = PB.posit_from_f64(torch.from_numpy(B64).cuda())
    C0 = PB.posit_from_f64(torch.from_numpy(C64).cuda())
for _ in range(2):
    C = C0.clone()
    PB.posit_gemm(A, B, C)
torch.cuda.synchronize()
print("ok")
