#!/bin/bash
# One long GPU-box call: the CPU oracle on the box's host cores for the largest
# configs (C4, C5p16) while the GPU runs the test suite and a bench;
# then the GPU outputs of those configs are compared with the fresh digests.
D=gpurun_out/r2a
mkdir -p $D
nproc > $D/nproc.txt; lscpu > $D/lscpu.txt 2>&1
OMP_NUM_THREADS=$(nproc) python tools/oracle_digests.py --configs C4,C5p16 \
   --out-dir $D/config_digests --cache /tmp/oracle_cache > $D/oracle.log 2>&1 &
OPID=$!
python tests/config_parity.py --configs C1 > $D/parity_c1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
python bench.py --steps 5 --warmup 3 > $D/bench.log 2>&1
wait $OPID; echo "oracle rc=$?" >> $D/oracle.log
python tests/config_parity.py --configs C4,C5p16 --digests $D/config_digests --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 python tests/config_parity.py --configs C4 --digests $D/config_digests --out $D/parity.jsonl >> $D/parity.log 2>&1
echo done
