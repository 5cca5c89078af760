#!/bin/bash
# quick look at one chunk call's results: bash tools/show_call.sh r2q1
D=gpurun_out/$1
for f in sum.log potf2_once.log factor.log gemm_variant_ab.log leaf_ab.log; do [ -f $D/$f ] && { echo "--- $f"; cat $D/$f; }; done
for f in parity.log parity_pcpack.log parity_bk32.log parity_leaf.log parity_serial.log parity_c4.log; do
  [ -f $D/$f ] && { echo "--- $f"; python - $D/$f <<'P'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        r = json.loads(l)
        print(r.get("config"), r.get("switches"), "OK" if r.get("ok") else r.get("skipped", "MISMATCH"), r.get("rows_compared", ""))
P
  }; done
echo "--- oracle"; tail -4 $D/oracle.log; cat $D/oracle_wait.log 2>/dev/null | tail -8
[ -f $D/pytest_gpu.log ] && tail -4 $D/pytest_gpu.log
[ -f $D/smoke.log ] && tail -2 $D/smoke.log
ls $D/config_digests 2>/dev/null
