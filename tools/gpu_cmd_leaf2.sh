T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/l2_tests_$T.log 2>&1; tail -n1 gpurun_out/l2_tests_$T.log
python tools/time_lapack.py --quick > gpurun_out/l2_time_$T.jsonl 2>&1
SWEEP_M=512,2048,8192 python tools/panel_sweep.py >> gpurun_out/l2_time_$T.jsonl 2>&1
echo done
