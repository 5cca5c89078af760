# launch lists: one LU panel step at n = 16384 (panel, laswp, TRSM) and a whole LU at n = 8192
T=${1:-rXX}
mkdir -p gpurun_out
python tools/prof_steps.py > gpurun_out/ps_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/steps_launches_$T.csv python tools/prof_steps.py > /dev/null 2>&1
python tools/prof_factor.py lu 8192 > gpurun_out/pf_lu8k_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu8k_launches_$T.csv python tools/prof_factor.py lu 8192 > /dev/null 2>&1
echo done
