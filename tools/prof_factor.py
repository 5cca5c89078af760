"""One posit_potrf or posit_getrf on a BASELINE recipe (for an ncu launch list).

    python tools/prof_factor.py chol 8192     # configs[2] recipe
    python tools/prof_factor.py lu 4096       # configs[3] recipe at n = 4096
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

kind, n = sys.argv[1], int(sys.argv[2])
info = torch.zeros(1, dtype=torch.int32, device="cuda")
if kind == "chol":
    A = PB.posit_from_f64(torch.from_numpy(SI.config3(n)).cuda())
    PB.posit_potrf(A, info, nb=256)
else:
    A = PB.posit_from_f64(torch.from_numpy(SI.config4(n)).cuda())
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    PB.posit_getrf(A, ipiv, info, nb=256)
torch.cuda.synchronize()
print("ok", int(info.cpu()[0]))
