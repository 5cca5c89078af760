#!/bin/bash
# r2q2: the evidence with the binary64-pipe division / sqrt opted in (decided from r2q1)
export POSIT_POTF2_DDIV=1 POSIT_LEAF_DDIV=1
bash tools/gpu_queue/evidence.sh $1
