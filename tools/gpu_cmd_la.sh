# lookahead A/B: tests with lookahead, then timings with POSIT_LOOKAHEAD=0 and =1 on the same box
mkdir -p gpurun_out
T=${1:-rXX}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$T.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_$T.log
POSIT_LOOKAHEAD=0 timeout 900 python tools/time_lapack.py > gpurun_out/lapack_${T}_la0.log 2>&1
POSIT_LOOKAHEAD=1 timeout 900 python tools/time_lapack.py > gpurun_out/lapack_${T}_la1.log 2>&1
echo done
