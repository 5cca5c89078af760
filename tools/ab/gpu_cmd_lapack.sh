# GPU parity tests + LU/Cholesky timing + ncu launch list of one LU panel step and a small Cholesky
T=${1:-rXX}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$T.log
timeout 900 python tools/time_lapack.py > gpurun_out/lapack_$T.log 2>&1; echo "exit $?" >> gpurun_out/lapack_$T.log
python tools/prof_steps.py > gpurun_out/steps_plain_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/steps_launches_$T.csv python tools/prof_steps.py > gpurun_out/steps_ncu_$T.log 2>&1
echo done
