T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pdl_tests_$T.log 2>&1; tail -n1 gpurun_out/pdl_tests_$T.log
for v in 1 0 1 0; do POSIT_PDL=$v TAG=pdl$v python tools/time_chol.py lu; POSIT_PDL=$v TAG=pdl$v python tools/time_chol.py chol; done > gpurun_out/pdl_time_$T.jsonl 2>&1
for v in 1 0; do POSIT_PDL=$v python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import synthetic_inputs as SI
from time_lapack import lu
lu('C4 pdl$v', SI.config4(), SI.C4_NB, reps=2)"; done >> gpurun_out/pdl_time_$T.jsonl 2>&1
python bench.py --no-cpu-baseline > gpurun_out/pdl_bench_$T.json 2>&1
echo done
