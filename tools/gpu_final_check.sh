#!/bin/bash
# Last check after a default flip that only moves a scheduling threshold: smoke, the LU / switch
# tests, every-word parity of the LU configs, timings and one bench line.
D=gpurun_out/${TAGDIR:-r2s}; mkdir -p $D
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 300 python tools/time_chol.py lu >> $D/factor.log 2>&1
timeout 300 python tools/time_chol.py c4 >> $D/factor.log 2>&1
timeout 300 python tools/time_chol.py chol >> $D/factor.log 2>&1
timeout 900 python tests/config_parity.py --configs C1,C5m16,C5m4,C5p0,C5p4,C5p16,C4 --out $D/parity.jsonl > $D/parity.log 2>&1
POSIT_LOOKAHEAD=0 POSIT_PDL=0 timeout 600 python tests/config_parity.py --configs C4 --out $D/parity_serial.jsonl > $D/parity_serial.log 2>&1
timeout 600 python -m pytest tests/test_gpu_lapack.py tests/test_gpu_switches.py -m gpu -q -p no:cacheprovider -k "getrf or lu or lapack_switches" > $D/pytest_lu.log 2>&1; echo "pytest rc=$? $(tail -1 $D/pytest_lu.log)" >> $D/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "bench rc=$?" >> $D/smoke.log
cat $D/smoke.log; grep -c '"ok": true' $D/parity.log $D/parity_serial.log; python - $D/factor.log <<'P'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        r = json.loads(l); print(f"{r['case']:30s} {r['ms']:9.2f} ms {r['gflops']:7.0f}")
P
