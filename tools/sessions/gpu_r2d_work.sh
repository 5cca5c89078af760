#!/bin/bash
# r2d: warp-per-row cluster potf2 (NC 8 / 16) and the chunked / 3-CTA Cholesky TRSM: correctness and timing
timeout 1200 python -m pytest tests/test_gpu_lapack.py tests/test_gpu_switches.py -m gpu -q -p no:cacheprovider -k "potrf or lapack_switches" > $D/pytest_potrf.log 2>&1; echo "pytest rc=$?" >> $D/pytest_potrf.log
BASE=paper_2401_14117_b200/ab/libposit_base.so
for v in "POSIT_POTF2=2" "POSIT_POTF2=2 POSIT_POTF2_NC=16" "POSIT_POTF2=1" "POSIT_RLTN=16,16,128" "POSIT_LIB_PATH=$BASE"; do
  env $v python tools/potf2_once.py >> $D/potf2_once.log 2>&1
  env $v TAG="$v" python tools/time_chol.py chol >> $D/chol_ab.log 2>&1
done
python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
POSIT_RLTN=16,16,128 python tools/chol_breakdown.py > $D/chol_breakdown_ch128.log 2>&1
python tests/config_parity.py --configs C3,C2,C1 > $D/parity_c3.log 2>&1
python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "bench rc=$?" >> $D/bench.log
