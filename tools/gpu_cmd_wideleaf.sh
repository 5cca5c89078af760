T=${1:-rXX}
mkdir -p gpurun_out
tail -n1 gpurun_out/wl_tests_r03t.log 2>/dev/null
for v in 4096 6144 16384 4096; do POSIT_WIDE_LEAF_COLS=$v TAG=wl$v python tools/time_chol.py lu; done > gpurun_out/wl_time_$T.jsonl 2>&1
for v in 4096 0; do POSIT_WIDE_LEAF_COLS=$v python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import synthetic_inputs as SI
from time_lapack import lu
lu('C4 wl$v', SI.config4(), SI.C4_NB, reps=2)"; done >> gpurun_out/wl_time_$T.jsonl 2>&1
echo done
