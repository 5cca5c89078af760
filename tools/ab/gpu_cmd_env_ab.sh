# A/B of an environment setting on C3 / C5 (alternating): gpu_cmd_env_ab.sh <tag> "<VAR=value>" "<workloads>"
T=${1:-rXX}; E=${2:-POSIT_GEMM_VARIANT=2}; W=${3:-chol}
mkdir -p gpurun_out
for i in 1 2; do
  for w in $W; do
    TAG=default python tools/time_chol.py $w
    env $E TAG="$E" python tools/time_chol.py $w
  done
done > gpurun_out/envab_$T.jsonl 2>&1
echo done
