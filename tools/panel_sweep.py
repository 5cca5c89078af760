"""Time posit_getrf_panel (nb = 256) for several heights m (run under gpurun;
POSIT_LEAF_CTAS selects the leaf configuration: 16 x 1024 or 148 x 256 threads)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402
from time_lapack import ev_time  # noqa: E402

for m in [int(x) for x in os.environ.get('SWEEP_M', '512,1024,2048,4096,8192,16384').split(',')]:
    P0 = PB.posit_from_f64(torch.from_numpy(SI.lu_matrix(m, 3)[:, :256].copy()).cuda())
    P = P0.clone()
    ipiv = torch.zeros(256, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    ms, _ = ev_time(lambda: (P.copy_(P0), PB.posit_getrf_panel(P, ipiv, info, 0)), warm=True)
    print(json.dumps({"m": m, "ctas": os.environ.get("POSIT_LEAF_CTAS", "default"), "panel_ms": ms}), flush=True)
