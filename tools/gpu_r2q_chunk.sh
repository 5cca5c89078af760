#!/bin/bash
# r2q: one <= 1 h call (gpurun clamps a call to 3600 s).  Host cores: the next chunk of
# the CPU oracle on configs[3] (C4, LU n = 16384), checkpointed in /tmp/c4ckpt every
# 8 min and at the budget, resumed by the next call if it lands on the same box; every
# checkpoint also writes C4_partial.json (digests of the rows already final).
# GPU meanwhile: $GPU_SCRIPT (A/Bs, evidence).  At the end: C4 parity against whatever
# digest exists (full or partial).
T=${TAGDIR:-r2q1}; D=gpurun_out/$T; mkdir -p $D $D/config_digests
NP=$(nproc); echo $NP > $D/nproc.txt
ls -la /tmp/c4ckpt > $D/ckpt_before.txt 2>&1
OB=${ORACLE_BUDGET:-3150}
OMP_NUM_THREADS=$NP nice -n 10 python tools/oracle_digests.py --configs C4 --out-dir $D/config_digests \
   --cache /tmp/oracle_cache --ckpt-dir /tmp/c4ckpt --time-budget $OB --ckpt-every 480 > $D/oracle.log 2>&1 &
OPID=$!
if [ -n "$GPU_SCRIPT" ]; then timeout 2400 bash $GPU_SCRIPT $D > $D/gpu_script.log 2>&1; fi
echo "gpu work done $(date)" >> $D/oracle_wait.log
wait $OPID; echo "oracle rc=$? $(date)" >> $D/oracle_wait.log
ls -la /tmp/c4ckpt >> $D/oracle_wait.log 2>&1
timeout 240 python tests/config_parity.py --configs C4 --digests $D/config_digests --out $D/parity_c4.jsonl > $D/parity_c4.log 2>&1
tail -3 $D/oracle.log; cut -c1-300 $D/parity_c4.log
