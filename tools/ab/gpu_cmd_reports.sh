# accuracy report + Table tabrandom analog (run after gpu_round.sh)
T=${1:-rXX}
mkdir -p gpurun_out
timeout 1200 python tools/accuracy_report.py --out gpurun_out/accuracy_$T.jsonl > gpurun_out/accuracy_$T.log 2>&1
timeout 600 python tools/op_microbench.py --out gpurun_out/op_microbench_$T.jsonl > gpurun_out/op_microbench_$T.log 2>&1
echo done
