T=${1:-rXX}
mkdir -p gpurun_out
for c in 16 148; do POSIT_LEAF_CTAS=$c python tools/panel_sweep.py; done > gpurun_out/panel_sweep_$T.jsonl 2>&1
echo done
