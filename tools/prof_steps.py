"""One LU panel step (n = 16384, nb = 256, step 0: panel, laswp, TRSM) and a
small Cholesky (n = 1024, nb = 256) for an ncu launch list of the panel-side
kernels (run under gpurun; the trailing GEMM is skipped to keep the list short).
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

n, nb = int(os.environ.get("PS_N", "16384")), 256
A = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(n, 3)).cuda())
ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
PB.posit_getrf_panel(A[:, :nb], ipiv[:nb], info, 0)
PB.posit_laswp(A[:, nb:], 0, nb, ipiv)
PB.posit_trsm("L", "L", "N", "U", A[:nb, :nb], A[:nb, nb:])
S = PB.posit_from_f64(torch.from_numpy(SI.config3(1024)).cuda())
PB.posit_potrf(S, info, nb=256)
torch.cuda.synchronize()
print("ok", int(info.cpu()[0]))
