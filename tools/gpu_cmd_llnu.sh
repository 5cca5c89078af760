# A/B of the LU TRSM in-block kernel (POSIT_LLNU_COL=8/4 thread-per-column row groups, 0 warp-per-column)
T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py tests/test_gpu_gemm.py -q -x > gpurun_out/llnu_tests_$T.log 2>&1; tail -3 gpurun_out/llnu_tests_$T.log
POSIT_LLNU_COL=4 python -m pytest tests/test_gpu_lapack.py -q -x -k "trsm or getrf" > gpurun_out/llnu_tests4_$T.log 2>&1; tail -1 gpurun_out/llnu_tests4_$T.log
for v in 8 4 0 8; do POSIT_LLNU_COL=$v python tools/time_lapack.py --quick > gpurun_out/llnu_time_${v}_$T.jsonl 2>&1; done
python tools/prof_steps.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/steps_launches_$T.csv python tools/prof_steps.py > /dev/null 2>&1
POSIT_LLNU_COL=4 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/steps_launches4_$T.csv python tools/prof_steps.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trsm_llnu_col -s 12 -c 1 -o gpurun_out/prof_llnu_$T python tools/prof_steps.py > gpurun_out/ncu_llnu_$T.log 2>&1
echo done
