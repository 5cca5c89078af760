#!/bin/bash
# The round's evidence on the library as built (plus whatever POSIT_* the caller exports):
# smoke, the full GPU suite, bench, factor timings and breakdowns, every-word parity at the
# default and the serial schedule, determinism, the ncu launch lists and full captures.
D=$1
env | grep '^POSIT_' > $D/env.txt
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
timeout 600 python tools/time_chol.py chol >> $D/factor.log 2>&1
timeout 600 python tools/time_chol.py lu >> $D/factor.log 2>&1
timeout 600 python tools/time_chol.py c4 >> $D/factor.log 2>&1
timeout 1800 python tests/config_parity.py --configs C1,C2,C3,C5m16,C5m4,C5p0,C5p4,C5p16 --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 timeout 1800 python tests/config_parity.py --configs C3,C5p0 --out $D/parity_serial.jsonl > $D/parity_serial.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 600 python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown.log 2>&1
LB_N=16384 timeout 900 python tools/lu_breakdown.py > $D/lu_breakdown_c4.log 2>&1
timeout 900 python tests/stress_determinism.py 10 > $D/determinism.log 2>&1
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-factor-keys"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $BCMD > $D/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_chol.csv python tools/prof_factor.py chol 8192 > $D/ncu_launch_chol.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_lu.csv python tools/prof_factor.py lu 8192 > $D/ncu_launch_lu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_d -s 1 -c 1 -o $D/prof_gemm_d python tools/prof_gemm.py > $D/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_potf2_cluster -s 3 -c 1 -o $D/prof_potf2 python tools/prof_factor.py chol 8192 > $D/ncu_potf2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_trsm_rltn_d -s 7 -c 1 -o $D/prof_rltn_d python tools/prof_factor.py chol 8192 > $D/ncu_rltn_d.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_leaf -s 40 -c 1 -o $D/prof_leaf python tools/prof_factor.py lu 8192 > $D/ncu_leaf.log 2>&1
tail -2 $D/smoke.log; tail -3 $D/pytest_gpu.log; cat $D/factor.log; grep -c '"ok": true' $D/parity.log
