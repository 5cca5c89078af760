#!/bin/bash
# r2q3: the evidence on the final library, no switches
bash tools/gpu_queue/evidence.sh $1
