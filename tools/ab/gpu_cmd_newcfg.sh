T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/nc_tests_$T.log 2>&1; tail -n1 gpurun_out/nc_tests_$T.log
python tools/tune_gemm.py 0 > gpurun_out/nc_tune_$T.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/nc_bench_$T.json 2>/dev/null
python tools/time_lapack.py --quick > gpurun_out/nc_time_$T.jsonl 2>&1
echo done
