# tiny GEMM path: all GPU tests, LU/Cholesky timings with and without it
T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/tiny_tests_$T.log 2>&1; tail -n1 gpurun_out/tiny_tests_$T.log
for v in 1; do POSIT_GEMM_TINY=$v python tools/time_lapack.py --quick > gpurun_out/tiny_time_${v}_$T.jsonl 2>&1; done
python tools/prof_factor.py lu 8192 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu8k_launches_$T.csv python tools/prof_factor.py lu 8192 > /dev/null 2>&1
echo done
