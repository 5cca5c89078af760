# A/B: current library vs variants/<name>.so on C5, C3 and C4 (alternating)
T=${1:-rXX}; V=${2:-nosplit}; W=${3:-lu chol}
mkdir -p gpurun_out
for i in 1 2; do
  for w in $W; do
    TAG=new python tools/time_chol.py $w
    POSIT_LIB_PATH=$PWD/paper_2401_14117_b200/variants/$V.so TAG=$V python tools/time_chol.py $w
  done
done > gpurun_out/ab_$T.jsonl 2>&1
echo done
