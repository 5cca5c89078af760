# A/B of several settings of one environment variable on C3 or C5, alternating:
# gpu_cmd_env_multi.sh <tag> <workload chol|lu> <VAR> <value> [<value> ...]  ("" = unset)
T=$1; W=$2; V=$3; shift 3
mkdir -p gpurun_out
for i in 1 2; do
  TAG=default python tools/time_chol.py $W
  for x in "$@"; do env $V="$x" TAG="$V=$x" python tools/time_chol.py $W; done
done > gpurun_out/envmulti_$T.jsonl 2>&1
echo done
