# A/B of the Cholesky TRSM variants (POSIT_RLTN="W,ROWS")
T=${1:-rXX}
mkdir -p gpurun_out
for v in 16,16 8,16 8,32 16,32; do
  POSIT_RLTN=$v python -m pytest tests/test_gpu_lapack.py -q -x -k "rltn or potrf or extreme" > gpurun_out/rltn_tests_${v}_$T.log 2>&1; echo "$v $(tail -n1 gpurun_out/rltn_tests_${v}_$T.log)"
done
for v in 16,16 8,16 8,32 16,16; do POSIT_RLTN=$v TAG=$v python tools/time_chol.py chol; done > gpurun_out/rltn_time_$T.jsonl 2>&1
echo done
