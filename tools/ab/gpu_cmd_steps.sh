mkdir -p gpurun_out
T=${1:-r01c}
python tools/prof_steps.py > gpurun_out/steps_plain_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/steps_launches_$T.csv python tools/prof_steps.py > gpurun_out/steps_ncu_$T.log 2>&1
echo done
