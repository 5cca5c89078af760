# GEMM change: the GEMM/LAPACK parity tests, bench line, lapack quick timings
T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/gc_tests_$T.log 2>&1; tail -n1 gpurun_out/gc_tests_$T.log
python bench.py --no-cpu-baseline > gpurun_out/gc_bench_$T.json 2>gpurun_out/gc_bench_$T.err
python tools/time_lapack.py --quick > gpurun_out/gc_lapack_$T.jsonl 2>&1
echo done
