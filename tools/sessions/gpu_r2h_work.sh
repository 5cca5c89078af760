#!/bin/bash
# r2h: the Cholesky TRSM and the tiny GEMM / SYRK on the D-MAC (default now),
# the GEMM table variants (product M in registers; 8-byte entries), timings.
mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 1200 python -m pytest tests/test_gpu_lapack.py tests/test_gpu_dmac.py tests/test_gpu_gemm.py -m gpu -q -x -p no:cacheprovider > $D/pytest.log 2>&1; echo "pytest rc=$?" >> $D/pytest.log
for v in "" "POSIT_LIB_PATH=paper_2401_14117_b200/ab/libposit_prodreg.so" "POSIT_LIB_PATH=paper_2401_14117_b200/ab/libposit_tab64.so" ""; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-factor-keys > $D/ab_tmp.log 2>&1
  echo "$v $(grep '^{' $D/ab_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms"], d["parity"]["mismatches"])')" >> $D/tab_ab.log
done
for p in 1 0; do
  POSIT_GEMM_PATH=$p TAG=path$p python tools/time_chol.py chol >> $D/factor.log 2>&1
done
TAG=d python tools/time_chol.py lu >> $D/factor.log 2>&1
TAG=d python tools/time_chol.py c4 >> $D/factor.log 2>&1
python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
timeout 900 python -m pytest tests/test_gpu_switches.py -m gpu -q -p no:cacheprovider > $D/pytest_sw.log 2>&1; echo "pytest rc=$?" >> $D/pytest_sw.log
python tests/config_parity.py --configs C3,C5m16,C5p0 > $D/parity.log 2>&1
