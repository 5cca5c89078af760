#!/bin/bash
# r2j: first check of the post-r2g library (D-MAC panel kernels): smoke,
# LU/Cholesky/D-MAC GPU tests, one bench line.
D=gpurun_out/r2j; mkdir -p $D
nproc > $D/nproc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python -m pytest tests/test_gpu_lapack.py tests/test_gpu_dmac.py -m gpu -q -x -p no:cacheprovider > $D/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $D/pytest_quick.log
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
tail -3 $D/pytest_quick.log; tail -2 $D/bench.log | cut -c1-600
