#!/bin/bash
# r2f: the binary64-pipe MAC (k_gemm_d): pipe rates, element and GEMM parity,
# bench both MAC paths, factorisation timings, one ncu capture of k_gemm_d.
mkdir -p $D
./tools/pipebench > $D/pipebench.json 2>&1
timeout 900 python -m pytest tests/test_gpu_dmac.py tests/test_gpu_gemm.py -m gpu -q -x -p no:cacheprovider > $D/pytest_d.log 2>&1; echo "pytest rc=$?" >> $D/pytest_d.log
timeout 900 python bench.py --steps 10 --warmup 3 > $D/bench_d.log 2>&1; echo "rc=$?" >> $D/bench_d.log
POSIT_GEMM_PATH=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_i.log 2>&1; echo "rc=$?" >> $D/bench_i.log
python tools/prof_gemm.py > $D/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_d -s 1 -c 1 -o $D/prof_gemm_d python tools/prof_gemm.py > $D/ncu_full.log 2>&1
for p in 1 0; do
  POSIT_GEMM_PATH=$p TAG=path$p python tools/time_chol.py chol >> $D/factor.log 2>&1
  POSIT_GEMM_PATH=$p TAG=path$p python tools/time_chol.py lu >> $D/factor.log 2>&1
done
POSIT_GEMM_PATH=1 TAG=path1 python tools/time_chol.py c4 >> $D/factor.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_switches.py -m gpu -q -p no:cacheprovider > $D/pytest_sw.log 2>&1; echo "pytest rc=$?" >> $D/pytest_sw.log
python tests/config_parity.py --configs C2,C3,C5p0,C1 > $D/parity.log 2>&1
