#!/bin/bash
# One GPU-box call (<= 1 h): a chunk of the resumable CPU oracle for the
# largest configs runs on the box's host cores in the background
# (checkpointed under /tmp/oracle_ckpt, which survives to the next call on
# the same box), while WORK_SCRIPT runs the GPU work of this call.  When the
# oracle finishes a config, its digest lands in gpurun_out/TAG/config_digests
# and the GPU output of that config is compared with it here.
#   bash tools/gpu_with_oracle.sh TAG BUDGET_S WORK_SCRIPT [CONFIGS]
TAG=$1; BUDGET=$2; WORK=$3; CFGS=${4:-C4,C5p16}
export D=gpurun_out/$TAG
mkdir -p $D
nproc > $D/nproc.txt
ls -la /tmp/oracle_ckpt > $D/ckpt_before.txt 2>&1
OMP_NUM_THREADS=$(( $(nproc) - 1 )) nice -n 19 python tools/oracle_digests.py --configs $CFGS --out-dir $D/config_digests \
    --cache /tmp/oracle_cache --ckpt-dir /tmp/oracle_ckpt --time-budget $BUDGET > $D/oracle.log 2>&1 &
OPID=$!
bash $WORK > $D/work.log 2>&1
echo "work rc=$?" >> $D/work.log
wait $OPID; echo "oracle rc=$?" >> $D/oracle.log
ls -la /tmp/oracle_ckpt >> $D/oracle.log 2>&1
for c in ${CFGS//,/ }; do
  if [ -f $D/config_digests/$c.json ]; then
    python tests/config_parity.py --configs $c --digests $D/config_digests --out $D/parity.jsonl >> $D/parity.log 2>&1
  fi
done
echo done
