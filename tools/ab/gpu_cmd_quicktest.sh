T=${1:-rXX}; K=${2:-getrf}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py -q -x -k "$K" > gpurun_out/qt_$T.log 2>&1; tail -n3 gpurun_out/qt_$T.log
POSIT_TAIL_W=0 python -m pytest tests/test_gpu_lapack.py -q -x -k "$K" > gpurun_out/qt0_$T.log 2>&1; tail -n1 gpurun_out/qt0_$T.log
echo done
