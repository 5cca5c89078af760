"""C3 Cholesky / C5 LU (median of 3) or C4 LU (median of 2) timing only, for A/B runs of panel-side variants:
    python tools/time_chol.py [chol|lu|c1|c4]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import synthetic_inputs as SI  # noqa: E402
from time_lapack import chol, lu  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "chol"
if which == "chol":
    chol("C3 " + os.environ.get("TAG", ""), SI.config3(), SI.C3_NB, reps=3)
elif which == "c1":
    lu("C1 " + os.environ.get("TAG", ""), SI.config1(), SI.C1_NB, reps=5)
elif which == "c4":
    lu("C4 " + os.environ.get("TAG", ""), SI.config4(), SI.C4_NB, reps=2)
else:
    lu("C5 s=0 " + os.environ.get("TAG", ""), SI.config5(0), SI.C5_NB, reps=3)
