# one compute-sanitizer tool per call: $1 tag, $2 tool (memcheck|racecheck|synccheck|initcheck)
mkdir -p gpurun_out
python tests/sanitize_small.py > gpurun_out/san_plain_$1.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $2 --print-limit 20 python tests/sanitize_small.py > gpurun_out/san_$2_$1.log 2>&1
echo "exit $?" >> gpurun_out/san_$2_$1.log
