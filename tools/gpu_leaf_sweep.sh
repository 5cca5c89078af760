#!/bin/bash
# Where the side-stream LU leaf should turn wide now that the trailing GEMM is 2.3x round 1's:
# POSIT_WIDE_LEAF_COLS (default 4096) x POSIT_SIDE_LEAF_CTAS x POSIT_LEAF_ROWS on C5 and C4.
D=gpurun_out/${TAGDIR:-r2r}; mkdir -p $D
for w in 4096 6144 8192; do
  for v in "" "POSIT_SIDE_LEAF_CTAS=16"; do
    env POSIT_WIDE_LEAF_COLS=$w $v TAG="wide=$w $v" timeout 200 python tools/time_chol.py lu >> $D/sweep.log 2>&1
  done
done
for w in 4096 8192; do
  for v in "" "POSIT_SIDE_LEAF_CTAS=32"; do
    env POSIT_WIDE_LEAF_COLS=$w $v TAG="wide=$w $v" timeout 200 python tools/time_chol.py c4 >> $D/sweep.log 2>&1
  done
done
python - $D/sweep.log <<'P'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        r = json.loads(l); print(f"{r['case']:70s} {r['ms']:9.2f} ms {r['gflops']:7.0f}")
P
