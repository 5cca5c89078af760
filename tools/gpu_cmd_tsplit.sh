T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/ts_tests_$T.log 2>&1; tail -n1 gpurun_out/ts_tests_$T.log
for v in 4096 0 4096; do POSIT_WIDE_LEAF_COLS=$v TAG=wl$v python tools/time_chol.py lu; done > gpurun_out/ts_time_$T.jsonl 2>&1
python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import synthetic_inputs as SI
from time_lapack import lu
lu('C4', SI.config4(), SI.C4_NB, reps=2)
lu('C1', SI.config1(), SI.C1_NB, reps=5)" >> gpurun_out/ts_time_$T.jsonl 2>&1
echo done
