mkdir -p gpurun_out
python tools/tune_gemm.py 0 1 2 3 5 > gpurun_out/tune_r01f.log 2>&1
./tools/pipebench > /dev/null 2>&1 && ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.sum -k regex:"kernILi(0|3|11|18|16|24|20|22)E" --csv ./tools/pipebench > gpurun_out/pipe_ncu.csv 2>&1
echo done
