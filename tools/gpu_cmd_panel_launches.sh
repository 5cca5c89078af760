T=${1:-rXX}
mkdir -p gpurun_out
SWEEP_M=512 python tools/panel_sweep.py > /dev/null 2>&1 && \
SWEEP_M=512 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/panel512_launches_$T.csv python tools/panel_sweep.py > /dev/null 2>&1
echo done
