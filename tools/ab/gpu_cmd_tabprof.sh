mkdir -p gpurun_out
T=${1:-rXX}
python tools/tabprof_analog.py --out gpurun_out/tabprof_$T.jsonl > gpurun_out/tabprof_$T.log 2>&1
python tools/tabprof_analog.py --count 1048576 --once > /dev/null 2>&1 && \
ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__sass_average_branch_targets_threads_uniform.pct,gpu__time_duration.sum --csv python tools/tabprof_analog.py --count 1048576 --once > gpurun_out/tabprof_ncu_$T.csv 2>&1
echo done
