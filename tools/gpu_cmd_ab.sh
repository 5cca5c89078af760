# A/B: current library vs variants/<name>.so on C5 and C4 (alternating)
T=${1:-rXX}; V=${2:-nosplit}
mkdir -p gpurun_out
for i in 1 2; do
  TAG=new python tools/time_chol.py lu
  POSIT_LIB_PATH=$PWD/paper_2401_14117_b200/variants/$V.so TAG=$V python tools/time_chol.py lu
done > gpurun_out/ab_$T.jsonl 2>&1
for L in "" "$PWD/paper_2401_14117_b200/variants/$V.so"; do POSIT_LIB_PATH=$L python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import synthetic_inputs as SI
from time_lapack import lu
lu('C4 ${L:+$V}', SI.config4(), SI.C4_NB, reps=2)"; done >> gpurun_out/ab_$T.jsonl 2>&1
echo done
