#!/bin/bash
# r2c: clean A/B of the Cholesky panel kernels (oracle now niced on n-1 cores)
for v in "POSIT_POTF2=2" "POSIT_POTF2=1" "POSIT_POTF2=2 POSIT_RLTN=16,16,0" "POSIT_POTF2=1 POSIT_RLTN=16,16,0"; do
  env $v TAG="$v" python tools/time_chol.py chol >> $D/chol_ab.log 2>&1
  env $v python tools/potf2_once.py >> $D/potf2_once.log 2>&1
done
python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
POSIT_RLTN=16,16,0 python tools/chol_breakdown.py > $D/chol_breakdown_lanes.log 2>&1
python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "bench rc=$?" >> $D/bench.log
