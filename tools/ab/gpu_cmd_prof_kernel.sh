# full ncu capture of one kernel launch: $1 tag, $2 kernel regex, $3 launches to skip, then the command
T=$1; K=$2; SKIP=$3; shift 3
mkdir -p gpurun_out
"$@" > gpurun_out/profk_plain_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/profk_$T "$@" > gpurun_out/profk_ncu_$T.log 2>&1
echo done
