T=${1:-rXX}
mkdir -p gpurun_out
for c in 4 8 16 32 64 148; do SWEEP_M=256,512,1024,2048,4096 POSIT_LEAF_CTAS=$c python tools/panel_sweep.py; done > gpurun_out/panel_sweep_$T.jsonl 2>&1
echo done
