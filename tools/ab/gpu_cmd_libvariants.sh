# time the GEMM shapes with each library variant under paper_2401_14117_b200/variants/ (default first and last)
mkdir -p gpurun_out
T=${1:-rXX}
python tools/tune_gemm.py 0 > gpurun_out/libvar_${T}_default.log 2>&1
for f in paper_2401_14117_b200/variants/*.so; do
  b=$(basename $f .so)
  POSIT_LIB_PATH=$PWD/$f python tools/tune_gemm.py 0 > gpurun_out/libvar_${T}_$b.log 2>&1
done
python tools/tune_gemm.py 0 > gpurun_out/libvar_${T}_default2.log 2>&1
echo done
