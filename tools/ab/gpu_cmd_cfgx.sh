T=${1:-rXX}
mkdir -p gpurun_out
POSIT_LIB_PATH=$PWD/paper_2401_14117_b200/variants/vx.so python tools/tune_gemm.py 0 8 7 14 15 10 1 3 6 > gpurun_out/cfgx_$T.log 2>&1
echo done
