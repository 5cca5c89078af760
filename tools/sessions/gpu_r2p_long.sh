#!/bin/bash
# r2p: one long call.  Host cores: the CPU oracle on configs[3] (C4, LU n = 16384,
# ~2.5 h on 16 cores) -> digests (or, if the budget runs out, the digests of the
# rows that are already final: C4_partial.json).  GPU meanwhile: the round's
# evidence on this library (smoke, full GPU suite, bench, breakdowns, every-word
# parity, ncu launch list + full captures).  At the end: C4 every-word parity.
D=gpurun_out/r2p; mkdir -p $D $D/config_digests
NP=$(nproc); echo $NP > $D/nproc.txt; lscpu > $D/lscpu.txt 2>&1
OB=${ORACLE_BUDGET:-10800}
OMP_NUM_THREADS=$NP nice -n 10 python tools/oracle_digests.py --configs C4 --out-dir $D/config_digests \
   --cache /tmp/oracle_cache --ckpt-dir /tmp/c4ckpt --time-budget $OB > $D/oracle.log 2>&1 &
OPID=$!
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
timeout 600 python tools/time_chol.py chol >> $D/factor.log 2>&1
timeout 600 python tools/time_chol.py lu >> $D/factor.log 2>&1
timeout 600 python tools/time_chol.py c4 >> $D/factor.log 2>&1
timeout 600 python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown.log 2>&1
LB_N=16384 timeout 900 python tools/lu_breakdown.py > $D/lu_breakdown_c4.log 2>&1
timeout 1800 python tests/config_parity.py --configs C1,C2,C3,C5m16,C5p0,C5p16 --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 timeout 1800 python tests/config_parity.py --configs C3,C5p0 --out $D/parity_serial.jsonl > $D/parity_serial.log 2>&1
timeout 900 python tests/stress_determinism.py 10 > $D/determinism.log 2>&1
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-factor-keys"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $BCMD > $D/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_chol.csv python tools/prof_factor.py chol 8192 > $D/ncu_launch_chol.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_lu.csv python tools/prof_factor.py lu 8192 > $D/ncu_launch_lu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_d -s 1 -c 1 -o $D/prof_gemm_d python tools/prof_gemm.py > $D/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_potf2_cluster -s 3 -c 1 -o $D/prof_potf2 python tools/prof_factor.py chol 8192 > $D/ncu_potf2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_trsm_rltn_d -s 7 -c 1 -o $D/prof_rltn_d python tools/prof_factor.py chol 8192 > $D/ncu_rltn_d.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_leaf -s 40 -c 1 -o $D/prof_leaf python tools/prof_factor.py lu 8192 > $D/ncu_leaf.log 2>&1
echo "gpu work done $(date)" >> $D/oracle_wait.log
wait $OPID; echo "oracle rc=$? $(date)" >> $D/oracle_wait.log
timeout 1200 python tests/config_parity.py --configs C4 --digests $D/config_digests --out $D/parity_c4.jsonl > $D/parity_c4.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 timeout 1200 python tests/config_parity.py --configs C4 --digests $D/config_digests --out $D/parity_c4.jsonl >> $D/parity_c4.log 2>&1
ls -la /tmp/c4ckpt >> $D/oracle_wait.log 2>&1
du -sh $D; echo done
