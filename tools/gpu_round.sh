#!/bin/bash
# One gpurun call: smoke, GPU parity tests, the bench line, LU/Cholesky timing,
# the ncu launch list of the bench command, and one full ncu capture of the GEMM kernel.
# usage: gpurun --timeout 2400 -- bash tools/gpu_round.sh <tag> [skip_ncu]
TAG=${1:-rXX}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench exit $?" >> gpurun_out/bench_$TAG.err
python bench.py --workload lu --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lu_$TAG.json 2> gpurun_out/bench_lu_$TAG.err
python bench.py --workload cholesky --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_chol_$TAG.json 2> gpurun_out/bench_chol_$TAG.err
timeout 900 python tools/time_lapack.py > gpurun_out/lapack_$TAG.log 2>&1
if [ "$2" != "skip_ncu" ]; then
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$BCMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $BCMD > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/prof_gemm.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 1 -c 1 -o gpurun_out/prof_gemm_$TAG python tools/prof_gemm.py > gpurun_out/ncu_full_$TAG.log 2>&1
# the first C4 trailing update (16128^2 x 256), SURVEY 8(d)
PROF_SHAPE=16128,16128,256 python tools/prof_gemm.py > gpurun_out/prof_plain_c4_$TAG.log 2>&1 && \
PROF_SHAPE=16128,16128,256 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 1 -c 1 -o gpurun_out/prof_gemm_c4_$TAG python tools/prof_gemm.py > gpurun_out/ncu_full_c4_$TAG.log 2>&1
fi
echo done
