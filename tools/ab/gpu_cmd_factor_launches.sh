T=${1:-rXX}
mkdir -p gpurun_out
python tools/prof_factor.py chol 8192 > gpurun_out/pf_chol_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_launches_$T.csv python tools/prof_factor.py chol 8192 > /dev/null 2>&1
python tools/prof_factor.py lu 4096 > gpurun_out/pf_lu_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu_launches_$T.csv python tools/prof_factor.py lu 4096 > /dev/null 2>&1
echo done
