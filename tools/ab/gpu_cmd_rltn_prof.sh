# ncu --set full of the first full-height Cholesky TRSM (k_trsm_rltn_fused, 496 CTAs at n = 8192)
T=${1:-rXX}
mkdir -p gpurun_out
python tools/prof_factor.py chol 8192 > gpurun_out/pf_chol_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trsm_rltn_fused -s 7 -c 1 -o gpurun_out/prof_rltn_$T python tools/prof_factor.py chol 8192 > gpurun_out/ncu_rltn_$T.log 2>&1
echo done
