T=${1:-rXX}
mkdir -p gpurun_out
for v in 16 8 4 16; do POSIT_SIDE_LEAF_CTAS=$v TAG=side$v python tools/time_chol.py lu; done > gpurun_out/sc_time_$T.jsonl 2>&1
for v in 16 8; do POSIT_SIDE_LEAF_CTAS=$v python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import synthetic_inputs as SI
from time_lapack import lu
lu('C4 side$v', SI.config4(), SI.C4_NB, reps=2)"; done >> gpurun_out/sc_time_$T.jsonl 2>&1
echo done
