T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/tt_tests_$T.log 2>&1; tail -n3 gpurun_out/tt_tests_$T.log
POSIT_TAIL_W=0 python -m pytest tests/test_gpu_lapack.py -q -x -k "getrf" > gpurun_out/tt_tests0_$T.log 2>&1; tail -n1 gpurun_out/tt_tests0_$T.log
echo done
