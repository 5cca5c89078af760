"""SHA-256 of posit_getrf's factors and pivots at configs[4] s = 0 (or LB_N):
compares a run-time schedule switch against the default on the GPU (the
default itself is checked against the oracle by tests/parity_report.py)."""
import hashlib
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

n = int(os.environ.get("LB_N", "8192"))
A = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(n, SI.C5_SEED)).cuda())
ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
PB.posit_getrf(A, ipiv, info, nb=256)
h = hashlib.sha256(A.cpu().numpy().tobytes() + ipiv.cpu().numpy().tobytes()).hexdigest()
print(n, int(info.cpu()[0]), h)
