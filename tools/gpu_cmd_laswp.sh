T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/lw_tests_$T.log 2>&1; tail -n1 gpurun_out/lw_tests_$T.log
python tools/time_lapack.py --quick > gpurun_out/lw_time_$T.jsonl 2>&1
python tools/prof_steps.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_laswp --csv --log-file gpurun_out/laswp_dram_$T.csv python tools/prof_steps.py > /dev/null 2>&1
echo done
