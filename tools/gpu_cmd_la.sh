# lookahead A/B: tests with lookahead forced on, then timings with POSIT_LOOKAHEAD=0 / default / 1 on the same box
mkdir -p gpurun_out
T=${1:-rXX}
POSIT_LOOKAHEAD=1 timeout 600 python -m pytest tests -q -m gpu -x -k "getrf or lapack or fullsize or dist or smoke or golden" > gpurun_out/pytest_gpu_$T.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_$T.log
POSIT_LOOKAHEAD=0 timeout 600 python tools/time_lapack.py > gpurun_out/lapack_${T}_la0.log 2>&1
timeout 600 python tools/time_lapack.py > gpurun_out/lapack_${T}_ladef.log 2>&1
POSIT_LOOKAHEAD=1 timeout 600 python tools/time_lapack.py > gpurun_out/lapack_${T}_la1.log 2>&1
echo done
