#!/bin/bash
# r2i: the D-MAC panel kernels (LU leaf, LU in-block solve g8, Cholesky TRSM,
# cluster potf2, tiny GEMM/SYRK): quick parity, bench, panel A/Bs,
# breakdowns, host-pipeline chunking, full GPU suite, ncu launch list.
mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python -m pytest tests/test_gpu_lapack.py tests/test_gpu_dmac.py -m gpu -q -x -p no:cacheprovider > $D/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $D/pytest_quick.log
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
for v in "" "POSIT_POTF2_NC=16" "POSIT_GEMM_PATH=0"; do env $v TAG="$v" python tools/time_chol.py chol >> $D/factor.log 2>&1; done
for v in "" "POSIT_LLNU_G8=0"; do env $v TAG="$v" python tools/time_chol.py lu >> $D/factor.log 2>&1; done
TAG=d python tools/time_chol.py c4 >> $D/factor.log 2>&1
for v in "" "POSIT_POTF2_NC=16"; do env $v python tools/potf2_once.py >> $D/potf2_once.log 2>&1; done
python tools/chol_breakdown.py > $D/chol_breakdown.log 2>&1
python tools/lu_breakdown.py > $D/lu_breakdown.log 2>&1
LB_N=16384 python tools/lu_breakdown.py > $D/lu_breakdown_c4.log 2>&1
for c in 2 4 8; do
  POSIT_HOST_CHUNKS=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-factor-keys > $D/ab_tmp.log 2>&1
  echo "chunks=$c $(grep '^{' $D/ab_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e"].get("parity"))')" >> $D/e2e_ab.log
done
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $BCMD > $D/ncu_launch.log 2>&1
