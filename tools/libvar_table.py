"""Table of tune_gemm.py results per library variant: python tools/libvar_table.py gpurun_out/libvar_<tag>_*.log"""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            cells = [f"{k.split()[0]}{'/' + k.split()[1] if len(k.split()) > 1 else ''}:{v['gflops']:.0f}"
                     for k, v in d.items() if isinstance(v, dict)]
            print(f.split("_")[-1].replace(".log", "").ljust(14), " ".join(cells[:6]))
