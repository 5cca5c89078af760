T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/c3t_tests_$T.log 2>&1; tail -n1 gpurun_out/c3t_tests_$T.log
for i in 1 2; do TAG=new python tools/time_chol.py chol; TAG=new python tools/time_chol.py lu; done > gpurun_out/c3t_time_$T.jsonl 2>&1
POSIT_LIB_PATH=$PWD/paper_2401_14117_b200/variants/base.so TAG=base python tools/time_chol.py chol >> gpurun_out/c3t_time_$T.jsonl 2>&1
python tools/prof_factor.py chol 8192 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_launches_$T.csv python tools/prof_factor.py chol 8192 > /dev/null 2>&1
echo done
