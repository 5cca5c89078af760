#!/bin/bash
# GPU side of r2q1: element tests and A/B of the binary64-pipe division / sqrt in the
# cluster potf2 (POSIT_POTF2_DDIV) and the LU leaf (POSIT_LEAF_DDIV).
D=$1
timeout 600 python -m pytest tests/test_gpu_dmac.py -m gpu -q -p no:cacheprovider > $D/pytest_dmac.log 2>&1; echo "dmac rc=$? $(tail -1 $D/pytest_dmac.log)" >> $D/sum.log
for v in "" "POSIT_POTF2_DDIV=1" "POSIT_POTF2_DDIV=1 POSIT_POTF2_NC=8" "POSIT_POTF2_DDIV=1 POSIT_POTF2_DEFER=1"; do
  echo "== $v" >> $D/potf2_once.log
  env $v timeout 120 python tools/potf2_once.py >> $D/potf2_once.log 2>&1 || echo "FAILED rc=$? ($v)" >> $D/potf2_once.log
done
for v in "" "POSIT_POTF2_DDIV=1" "POSIT_POTF2_DDIV=1 POSIT_POTF2_DEFER=1"; do env $v TAG="$v" timeout 300 python tools/time_chol.py chol >> $D/factor.log 2>&1; done
for v in "" "POSIT_LEAF_DDIV=1"; do env $v TAG="$v" timeout 300 python tools/time_chol.py lu >> $D/factor.log 2>&1; done
for v in "" "POSIT_LEAF_DDIV=1"; do env $v TAG="$v" timeout 300 python tools/time_chol.py c4 >> $D/factor.log 2>&1; done
for v in "POSIT_POTF2_DDIV=1" "POSIT_LEAF_DDIV=1" "POSIT_POTF2_DDIV=1 POSIT_LEAF_DDIV=1"; do
  env $v timeout 900 python -m pytest tests/test_gpu_lapack.py -m gpu -q -p no:cacheprovider > $D/pytest_lapack.log 2>&1; echo "lapack [$v] rc=$? $(tail -1 $D/pytest_lapack.log)" >> $D/sum.log
done
timeout 900 python -m pytest tests/test_gpu_switches.py -m gpu -q -p no:cacheprovider -k "lapack_switches and (POTF2 or LEAF_DDIV)" > $D/pytest_sw.log 2>&1; echo "switches rc=$? $(tail -1 $D/pytest_sw.log)" >> $D/sum.log
POSIT_POTF2_DDIV=1 timeout 600 python tests/config_parity.py --configs C3 --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LEAF_DDIV=1 timeout 900 python tests/config_parity.py --configs C1,C5m16,C5p0,C5p16 --out $D/parity.jsonl >> $D/parity.log 2>&1
POSIT_POTF2_DDIV=1 timeout 600 python tools/chol_breakdown.py > $D/chol_breakdown_ddiv.log 2>&1
POSIT_LEAF_DDIV=1 timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown_ddiv.log 2>&1
POSIT_POTF2_DDIV=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potf2_cluster -s 3 -c 1 -o $D/prof_potf2_ddiv python tools/prof_factor.py chol 8192 > $D/ncu_potf2.log 2>&1
# the packed column buffer (-DPC_PACKED=1) as a second library
V=$PWD/paper_2401_14117_b200/ab/libposit_pcpack.so
if [ -f $V ]; then
  for v in "" "POSIT_POTF2_DDIV=1" "POSIT_POTF2_DDIV=1 POSIT_POTF2_NC=8"; do
    echo "== pcpack $v" >> $D/potf2_once.log
    env POSIT_LIB_PATH=$V $v timeout 120 python tools/potf2_once.py >> $D/potf2_once.log 2>&1 || echo "FAILED rc=$? (pcpack $v)" >> $D/potf2_once.log
  done
  for v in "" "POSIT_POTF2_DDIV=1"; do env POSIT_LIB_PATH=$V $v TAG="pcpack $v" timeout 300 python tools/time_chol.py chol >> $D/factor.log 2>&1; done
  for v in "" "POSIT_POTF2_DDIV=1"; do
    env POSIT_LIB_PATH=$V $v timeout 900 python -m pytest tests/test_gpu_lapack.py -m gpu -q -p no:cacheprovider -k "potrf or chol or potf2" > $D/pytest_pcpack.log 2>&1; echo "pcpack lapack [$v] rc=$? $(tail -1 $D/pytest_pcpack.log)" >> $D/sum.log
    env POSIT_LIB_PATH=$V $v timeout 600 python tests/config_parity.py --configs C3 --out $D/parity_pcpack.jsonl >> $D/parity_pcpack.log 2>&1
  done
fi
# GEMM tile A/B on C2 (D1 64x128 / 1024 threads / 1 CTA per SM is the model's choice; r2m ncu: 7 % of the
# stall samples at the slab barrier): D2 64x64, D3 32x128, D4 128x32 with 512 threads, 2 CTAs per SM
for v in 21 22 23 24; do
  POSIT_GEMM_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-factor-keys > $D/ab_tmp.log 2>&1
  echo "variant=$v $(grep '^{' $D/ab_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["parity"]["mismatches"])')" >> $D/gemm_variant_ab.log
done
# k-slab depth 32 (half the CTA barriers) as a second library
V2=$PWD/paper_2401_14117_b200/ab/libposit_bk32.so
if [ -f $V2 ]; then
  for v in 21 22; do
    POSIT_LIB_PATH=$V2 POSIT_GEMM_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-factor-keys > $D/ab_tmp.log 2>&1
    echo "bk32 variant=$v $(grep '^{' $D/ab_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["parity"]["mismatches"])')" >> $D/gemm_variant_ab.log
  done
  POSIT_LIB_PATH=$V2 TAG=bk32 timeout 300 python tools/time_chol.py chol >> $D/factor.log 2>&1
  POSIT_LIB_PATH=$V2 TAG=bk32 timeout 300 python tools/time_chol.py lu >> $D/factor.log 2>&1
  POSIT_LIB_PATH=$V2 TAG=bk32 timeout 300 python tools/time_chol.py c4 >> $D/factor.log 2>&1
  POSIT_LIB_PATH=$V2 timeout 900 python -m pytest tests/test_gpu_gemm.py -m gpu -q -p no:cacheprovider > $D/pytest_bk32.log 2>&1; echo "bk32 gemm tests rc=$? $(tail -1 $D/pytest_bk32.log)" >> $D/sum.log
  POSIT_LIB_PATH=$V2 timeout 900 python tests/config_parity.py --configs C2,C3,C5p0 --out $D/parity_bk32.jsonl > $D/parity_bk32.log 2>&1
fi
cat $D/sum.log $D/potf2_once.log $D/factor.log $D/gemm_variant_ab.log
