# diagonal-block Cholesky variants (POSIT_POTF2=1 blocked + tiny SYRK, 0 recursive): parity, C3 timing, launches
T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py -q -x > gpurun_out/potf2_tests_$T.log 2>&1; tail -n1 gpurun_out/potf2_tests_$T.log
python -m pytest tests/test_gpu_fullsize.py -q -x -k "cholesky" > gpurun_out/potf2_full_$T.log 2>&1; tail -n1 gpurun_out/potf2_full_$T.log
for v in 1 0 1; do POSIT_POTF2=$v TAG=potf2_$v python tools/time_chol.py chol; done > gpurun_out/potf2_time_$T.jsonl 2>&1
python tools/prof_factor.py chol 8192 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_launches_$T.csv python tools/prof_factor.py chol 8192 > /dev/null 2>&1
echo done
