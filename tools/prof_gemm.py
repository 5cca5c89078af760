"""One warm-up + one profiled posit_gemm launch on configs[1] (for ncu)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

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
