"""C3 Cholesky timing only (median of 3), for A/B runs of panel-side variants."""
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
else:
    lu("C5 s=0 " + os.environ.get("TAG", ""), SI.config5(0), SI.C5_NB, reps=3)
