#!/bin/bash
# r2k: one long call.  Host cores: the CPU oracle on configs[3] (C4, LU
# n = 16384, ~2.5 h) -> digests, checkpointed to /tmp if the budget runs out.
# GPU meanwhile: full GPU suite, bench, panel A/Bs, breakdowns, e2e chunking,
# ncu launch list and full captures (GEMM, Cholesky TRSM, cluster potf2),
# every-word parity of C1/C2/C3/C5 at default switches and serial schedule.
# At the end: C4 every-word parity against the fresh digests.
D=gpurun_out/r2k; mkdir -p $D $D/config_digests
NP=$(nproc); echo $NP > $D/nproc.txt; lscpu > $D/lscpu.txt 2>&1
OB=${ORACLE_BUDGET:-10800}
OMP_NUM_THREADS=$((NP-1)) nice -n 19 python tools/oracle_digests.py --configs C4 --out-dir $D/config_digests \
   --cache /tmp/oracle_cache --ckpt-dir /tmp/c4ckpt --time-budget $OB > $D/oracle.log 2>&1 &
OPID=$!
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
for v in "" "POSIT_POTF2_NC=16" "POSIT_GEMM_PATH=0"; do env $v TAG="$v" timeout 600 python tools/time_chol.py chol >> $D/factor.log 2>&1; done
for v in "" "POSIT_LLNU_G8=0"; do env $v TAG="$v" timeout 600 python tools/time_chol.py lu >> $D/factor.log 2>&1; done
TAG=d timeout 600 python tools/time_chol.py c4 >> $D/factor.log 2>&1
for v in "" "POSIT_POTF2_NC=16"; do env $v timeout 300 python tools/potf2_once.py >> $D/potf2_once.log 2>&1; done
timeout 600 python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown.log 2>&1
LB_N=16384 timeout 900 python tools/lu_breakdown.py > $D/lu_breakdown_c4.log 2>&1
for c in 2 4 8; do
  POSIT_HOST_CHUNKS=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-factor-keys > $D/ab_tmp.log 2>&1
  echo "chunks=$c $(grep '^{' $D/ab_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e"].get("parity"))')" >> $D/e2e_ab.log
done
timeout 1800 python tests/config_parity.py --configs C1,C2,C3,C5m16,C5p0,C5p16 --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 timeout 1800 python tests/config_parity.py --configs C3,C5p0 --out $D/parity.jsonl >> $D/parity.log 2>&1
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $BCMD > $D/ncu_launch.log 2>&1
python tools/prof_gemm.py > $D/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_d -s 1 -c 1 -o $D/prof_gemm_d python tools/prof_gemm.py > $D/ncu_gemm.log 2>&1
python tools/prof_factor.py chol 8192 > $D/pf_chol.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trsm_rltn_fused -s 7 -c 1 -o $D/prof_rltn python tools/prof_factor.py chol 8192 > $D/ncu_rltn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_potf2_cluster -s 3 -c 1 -o $D/prof_potf2 python tools/prof_factor.py chol 8192 > $D/ncu_potf2.log 2>&1
echo "gpu work done $(date)" >> $D/oracle_wait.log
wait $OPID; echo "oracle rc=$? $(date)" >> $D/oracle_wait.log
if [ -f $D/config_digests/C4.json ]; then
  timeout 1200 python tests/config_parity.py --configs C4 --digests $D/config_digests --out $D/parity_c4.jsonl > $D/parity_c4.log 2>&1
fi
ls -la /tmp/c4ckpt >> $D/oracle_wait.log 2>&1
echo done
