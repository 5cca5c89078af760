"""Instruction mix per MAC of the hot loops of one kernel in a SASS dump
(marker: one DFMA per D-MAC, or FLO per integer MAC).
    python tools/sass_loop.py <sass-file-or-.so/.o> <kernel-substring> [DFMA|FLO]"""
import collections
import re
import subprocess
import sys

src, pat = sys.argv[1], sys.argv[2]
mark = sys.argv[3] if len(sys.argv) > 3 else "DFMA"
txt = open(src).read() if src.endswith(".sass") else subprocess.run(["cuobjdump", "-sass", src], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt):
    name = f.split("\n")[0]
    if pat not in name:
        continue
    ins = [(int(m.group(1), 16), m.group(2).strip()) for l in f.split("\n") for m in [re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)] if m]
    for a, t in ins:
        m = re.search(r"BRA.*?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            body = [x[1] for x in ins if int(m.group(1), 16) <= x[0] <= a]
            n = sum(1 for x in body if x.startswith(mark))
            if n == 0 or len(body) > 2000:
                continue
            c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
            print(f"{name.strip()[:70]} loop {len(body)} / {n} MACs = {len(body) / n:.2f} per MAC")
            print("   ", ", ".join(f"{k} {v / n:.2f}" for k, v in sorted(c.items(), key=lambda x: -x[1])))
    break
