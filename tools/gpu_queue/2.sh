#!/bin/bash
# r2q2: A/B of the LU leaf's row-mode update (POSIT_LEAF_ROWS) on the library as rebuilt after
# r2q1's A/B, then the evidence on that library.
D=$1
for v in "" "POSIT_LEAF_ROWS=1" "POSIT_LEAF_ROWS=1 POSIT_LEAF_DDIV=1" "POSIT_LEAF_DDIV=1"; do env $v TAG="$v" timeout 300 python tools/time_chol.py lu >> $D/leaf_ab.log 2>&1; done
for v in "" "POSIT_LEAF_ROWS=1 POSIT_LEAF_DDIV=1"; do env $v TAG="$v" timeout 300 python tools/time_chol.py c4 >> $D/leaf_ab.log 2>&1; done
POSIT_LEAF_ROWS=1 POSIT_LEAF_DDIV=1 timeout 900 python tests/config_parity.py --configs C1,C5m16,C5p0,C5p16 --out $D/parity_leaf.jsonl > $D/parity_leaf.log 2>&1
POSIT_LEAF_ROWS=1 POSIT_LEAF_DDIV=1 timeout 600 python -m pytest tests/test_gpu_lapack.py -m gpu -q -p no:cacheprovider -k "getrf or lu or trsm" > $D/pytest_leaf.log 2>&1; echo "leaf rows+ddiv lapack rc=$? $(tail -1 $D/pytest_leaf.log)" >> $D/leaf_ab.log
POSIT_LEAF_ROWS=1 POSIT_LEAF_DDIV=1 timeout 600 python tools/lu_breakdown.py > $D/lu_breakdown_leafrows.log 2>&1
POSIT_LEAF_ROWS=1 POSIT_LEAF_DDIV=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_lu_leafrows.csv python tools/prof_factor.py lu 8192 > $D/ncu_launch_lu_leafrows.log 2>&1
cat $D/leaf_ab.log
bash tools/gpu_queue/evidence.sh $1
