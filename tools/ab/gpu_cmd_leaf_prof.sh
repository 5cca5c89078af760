# ncu --set full of one cooperative LU leaf (first leaf of the n = 16384 panel, 148 CTAs)
T=${1:-rXX}
mkdir -p gpurun_out
python tools/prof_steps.py > gpurun_out/ps_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_leaf_coop -s 0 -c 1 -o gpurun_out/prof_leaf_$T python tools/prof_steps.py > gpurun_out/ncu_leaf_$T.log 2>&1
echo done
