# ncu --set full of one diagonal-block Cholesky leaf (k_potf2_leaf)
T=${1:-rXX}
mkdir -p gpurun_out
python tools/prof_factor.py chol 1024 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_potf2_leaf -s 2 -c 1 -o gpurun_out/prof_potf2_$T python tools/prof_factor.py chol 1024 > gpurun_out/ncu_potf2_$T.log 2>&1
echo done
