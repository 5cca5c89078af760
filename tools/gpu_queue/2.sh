#!/bin/bash
# r2q2: the evidence on the library as rebuilt after r2q1's A/B (defaults flipped in the sources)
bash tools/gpu_queue/evidence.sh $1
