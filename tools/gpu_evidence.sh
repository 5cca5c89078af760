# evidence refresh without the round script: reports (accuracy, op microbench, tabprof), parity, determinism, paper figures
T=${1:-rXX}
mkdir -p gpurun_out
bash tools/gpu_cmd_reports.sh $T
timeout 1500 python tests/parity_report.py --out gpurun_out/parity_report_$T.json > gpurun_out/parity_report_$T.log 2>&1
timeout 900 python tests/stress_determinism.py 10 > gpurun_out/stress_$T.log 2>&1
timeout 900 python tools/paper_figures.py --out gpurun_out/paper_figures_$T.jsonl > gpurun_out/paper_figures_$T.log 2>&1
echo done
