# end-of-round evidence: round script (smoke, tests, bench, timings, ncu), reports, parity, determinism
T=${1:-rXX}
bash tools/gpu_round.sh $T
bash tools/gpu_cmd_reports.sh $T
timeout 1500 python tests/parity_report.py --out gpurun_out/parity_report_$T.json > gpurun_out/parity_report_$T.log 2>&1
timeout 900 python tests/stress_determinism.py 10 > gpurun_out/stress_$T.log 2>&1
timeout 900 python tools/paper_figures.py --out gpurun_out/paper_figures_$T.jsonl > gpurun_out/paper_figures_$T.log 2>&1
echo done
