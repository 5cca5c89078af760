#!/bin/bash
# r2n/r2o: sanity + A/B of the deferred-update cluster potf2 before the long call.
D=gpurun_out/${TAGDIR:-r2o}; mkdir -p $D
for v in "" "POSIT_POTF2_DEFER=1" "POSIT_POTF2_DEFER=2" "POSIT_POTF2_NC=8" "POSIT_POTF2_NC=8 POSIT_POTF2_DEFER=2"; do
  echo "== $v" >> $D/potf2_once.log
  env $v timeout 120 python tools/potf2_once.py >> $D/potf2_once.log 2>&1 || echo "FAILED rc=$? ($v)" >> $D/potf2_once.log
done
for v in "" "POSIT_POTF2_DEFER=2"; do env $v TAG="$v" timeout 300 python tools/time_chol.py chol >> $D/factor.log 2>&1; done
for v in "" "POSIT_POTF2_DEFER=1" "POSIT_POTF2_DEFER=2"; do
env $v timeout 900 python -m pytest tests/test_gpu_lapack.py -m gpu -q -p no:cacheprovider -k "potrf or chol or potf2" > $D/pytest_chol.log 2>&1; echo "pytest [$v] rc=$? $(tail -1 $D/pytest_chol.log)" >> $D/pytest_sum.log
done
timeout 900 python -m pytest tests/test_gpu_switches.py -m gpu -q -p no:cacheprovider -k "lapack_switches and POTF2" > $D/pytest_sw.log 2>&1; echo "pytest switches rc=$? $(tail -1 $D/pytest_sw.log)" >> $D/pytest_sum.log
POSIT_POTF2_DEFER=2 timeout 600 python tests/config_parity.py --configs C3 --out $D/parity.jsonl > $D/parity.log 2>&1
cat $D/potf2_once.log $D/factor.log $D/pytest_sum.log; cut -c1-250 $D/parity.log
