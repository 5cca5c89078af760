T=${1:-rXX}
mkdir -p gpurun_out
for v in 512 256 384 768 0 512; do POSIT_TAIL_W=$v TAG=tail$v python tools/time_chol.py lu; done > gpurun_out/tail_time_$T.jsonl 2>&1
for v in 256 512 0; do POSIT_TAIL_W=$v python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import synthetic_inputs as SI
from time_lapack import lu
lu('C4 tail$v', SI.config4(), SI.C4_NB, reps=2)"; done >> gpurun_out/tail_time_$T.jsonl 2>&1
echo done
