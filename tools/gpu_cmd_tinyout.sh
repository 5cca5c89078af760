T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/to_tests_$T.log 2>&1; tail -n1 gpurun_out/to_tests_$T.log
for v in 65536 0 16384 262144; do POSIT_TINY_OUTPUTS=$v SWEEP_M=512,2048 python tools/panel_sweep.py; POSIT_TINY_OUTPUTS=$v TAG=to$v python tools/time_chol.py lu; POSIT_TINY_OUTPUTS=$v TAG=to$v python tools/time_chol.py chol; done > gpurun_out/to_time_$T.jsonl 2>&1
echo done
