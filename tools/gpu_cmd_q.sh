mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k 'trsm or potrf or golden or smoke' > gpurun_out/pytest_gpu_r01q.log 2>&1
for w in 8 16; do POSIT_RLTN_W=$w python tools/prof_factor.py chol 8192 > /dev/null 2>&1 && POSIT_RLTN_W=$w ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_launches_r01q_w$w.csv python tools/prof_factor.py chol 8192 > /dev/null 2>&1; done
POSIT_RLTN_W=16 timeout 900 python tools/time_lapack.py --quick > gpurun_out/lapack_r01q.log 2>&1
