#!/bin/bash
# Local driver: back-to-back <= 1 h gpurun calls, each running the next chunk of the C4
# oracle (tools/gpu_r2q_chunk.sh) plus tools/gpu_queue/<i>.sh on the GPU, until the full
# digest exists or $2 calls are done.  Retries while another call is in flight.
START=${1:-1}; END=${2:-3}
for i in $(seq $START $END); do
  T=r2q$i
  # between calls: up to ${GO_WAIT:-230} s for the operator to read the last call's results and
  # prepare this call's queue script / defaults (touch /tmp/go_$i to start at once); the box is
  # kept for 5 min after a call, and the oracle checkpoint lives in its /tmp
  if [ $i -gt $START ]; then
    w=0; while [ ! -f /tmp/go_$i ] && [ $w -lt ${GO_WAIT:-230} ]; do sleep 2; w=$((w+2)); done
  fi
  GS=""; [ -f tools/gpu_queue/$i.sh ] && GS=tools/gpu_queue/$i.sh
  while true; do
    gpurun --timeout 3600 -- "TAGDIR=$T GPU_SCRIPT=$GS ORACLE_BUDGET=${OB:-3250} bash tools/gpu_r2q_chunk.sh" > /tmp/chunk_$T.log 2>&1
    rc=$?
    if grep -q "status=ok\|merged" /tmp/chunk_$T.log; then break; fi
    echo "call $T refused or failed (rc=$rc), retrying in 20 s: $(tail -1 /tmp/chunk_$T.log)" >> /tmp/chunk_loop.log
    sleep 20
  done
  echo "call $T done $(date): $(tail -2 /tmp/chunk_$T.log | head -1)" >> /tmp/chunk_loop.log
  if [ -f gpurun_out/$T/config_digests/C4.json ]; then echo "C4 digest complete after $T" >> /tmp/chunk_loop.log; break; fi
done
echo "loop finished $(date)" >> /tmp/chunk_loop.log
