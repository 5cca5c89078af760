mkdir -p gpurun_out
T=${1:-rXX}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$T.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_$T.log
timeout 900 python tools/time_lapack.py > gpurun_out/lapack_$T.log 2>&1
bash tools/gpu_cmd_factor_launches.sh $T
