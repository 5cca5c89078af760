#!/bin/bash
# r2m: evidence for the final round-2 library + A/B of the opt-in D-MAC TRSMs.
D=gpurun_out/r2m; mkdir -p $D
nproc > $D/nproc.txt; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $D/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
# A/B first (cheap, decides defaults)
for v in "" "POSIT_RLTN_D=1" "POSIT_RLTN_D=1 POSIT_POTF2_NC=16" "POSIT_POTF2_NC=16"; do env $v TAG="$v" timeout 600 python tools/time_chol.py chol >> $D/factor.log 2>&1; done
for v in "" "POSIT_LLNU_D=1" "POSIT_LLNU_G8=0"; do env $v TAG="$v" timeout 600 python tools/time_chol.py lu >> $D/factor.log 2>&1; done
for v in "" "POSIT_LLNU_D=1"; do env $v TAG="$v" timeout 600 python tools/time_chol.py c4 >> $D/factor.log 2>&1; done
POSIT_RLTN_D=1 timeout 900 python tests/config_parity.py --configs C3 --out $D/parity_optin.jsonl > $D/parity_optin.log 2>&1
POSIT_LLNU_D=1 timeout 1200 python tests/config_parity.py --configs C1,C5m16,C5p0,C5p16 --out $D/parity_optin.jsonl >> $D/parity_optin.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 1800 python tests/config_parity.py --configs C1,C2,C3,C5m16,C5p0,C5p16,C4 --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 timeout 1800 python tests/config_parity.py --configs C3,C5p0 --out $D/parity_serial.jsonl > $D/parity_serial.log 2>&1
timeout 600 python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
POSIT_RLTN_D=1 timeout 600 python tools/chol_breakdown.py > $D/chol_breakdown_rltn_d.log 2>&1
timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown.log 2>&1
POSIT_LLNU_D=1 timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown_llnu_d.log 2>&1
LB_N=16384 timeout 900 python tools/lu_breakdown.py > $D/lu_breakdown_c4.log 2>&1
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-factor-keys"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $BCMD > $D/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_chol.csv python tools/prof_factor.py chol 8192 > $D/ncu_launch_chol.log 2>&1
python tools/prof_gemm.py > $D/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_d -s 1 -c 1 -o $D/prof_gemm_d python tools/prof_gemm.py > $D/ncu_gemm.log 2>&1
python tools/prof_factor.py chol 8192 > $D/pf_chol.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_trsm_rltn_fused -s 7 -c 1 -o $D/prof_rltn python tools/prof_factor.py chol 8192 > $D/ncu_rltn.log 2>&1
POSIT_RLTN_D=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trsm_rltn_d -s 7 -c 1 -o $D/prof_rltn_d python tools/prof_factor.py chol 8192 > $D/ncu_rltn_d.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_potf2_cluster -s 3 -c 1 -o $D/prof_potf2 python tools/prof_factor.py chol 8192 > $D/ncu_potf2.log 2>&1
ls -la $D; du -sh $D
echo done
