# host-pipelined GEMM: parity test, bench (e2e) with pipeline on and off
T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/host_tests_$T.log 2>&1; tail -n1 gpurun_out/host_tests_$T.log
python bench.py --no-cpu-baseline > gpurun_out/host_bench1_$T.json 2>&1
POSIT_HOST_PIPELINE=0 python bench.py --no-cpu-baseline > gpurun_out/host_bench0_$T.json 2>&1
echo done
