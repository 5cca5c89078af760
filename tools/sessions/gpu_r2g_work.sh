#!/bin/bash
# r2g: the binary64-pipe GEMM as the default: the shared-table layout A/B
# (4-byte entries vs 8-byte, both sign-folded), full GPU suite, bench,
# breakdowns, the bench's ncu launch list, one ncu capture of k_gemm_d.
mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
for v in "" "POSIT_LIB_PATH=paper_2401_14117_b200/ab/libposit_tab64.so" ""; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-factor-keys > $D/ab_tmp.log 2>&1
  echo "$v $(grep '^{' $D/ab_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms"], d["parity"]["mismatches"])')" >> $D/tab_ab.log
done
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
python tools/prof_gemm.py > $D/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_d -s 1 -c 1 -o $D/prof_gemm_d python tools/prof_gemm.py > $D/ncu_full.log 2>&1
python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
python tools/lu_breakdown.py > $D/lu_breakdown.log 2>&1
LB_N=16384 python tools/lu_breakdown.py > $D/lu_breakdown_c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
