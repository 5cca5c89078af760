# panel leaf change: parity (lapack + full-size LU tests), timings, leaf ncu
T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lapack.py tests/test_gpu_dist.py -q -x > gpurun_out/leaf_tests_$T.log 2>&1; tail -n1 gpurun_out/leaf_tests_$T.log
python -m pytest tests/test_gpu_fullsize.py -q -x -k "lu" > gpurun_out/leaf_full_$T.log 2>&1; tail -n1 gpurun_out/leaf_full_$T.log
for v in 1 2 1; do POSIT_LEAF_COOP=$v python tools/time_lapack.py --quick > gpurun_out/leaf_time_${v}_$T.jsonl 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:k_leaf_coop -s 0 -c 1 -o gpurun_out/prof_leaf_$T python tools/prof_steps.py > gpurun_out/ncu_leaf_$T.log 2>&1
echo done
