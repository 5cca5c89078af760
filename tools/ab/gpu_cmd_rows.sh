mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "trsm or potrf or fullsize" > gpurun_out/pytest_rows.log 2>&1; echo "exit $?" >> gpurun_out/pytest_rows.log
for r in 16 32; do POSIT_RLTN_ROWS=$r timeout 600 python tools/time_lapack.py --quick > gpurun_out/lapack_rows$r.log 2>&1; done
for r in 16 32; do POSIT_RLTN_ROWS=$r python tools/prof_factor.py chol 8192 >/dev/null 2>&1 && POSIT_RLTN_ROWS=$r POSIT_LOOKAHEAD=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_rows$r.csv python tools/prof_factor.py chol 8192 > /dev/null 2>&1; done
