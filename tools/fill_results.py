"""Rewrite the round-2 results tables of README.md and DESIGN.md (between the R2_TABLE markers)
from one evidence tag under profiles/ (written by tools/evidence_to_profiles.py).

    python tools/fill_results.py r2q3
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
P = os.path.join(ROOT, "profiles")
b = json.loads(open(os.path.join(P, f"{tag}_bench.json")).readline())
fac = {}
for l in open(os.path.join(P, f"{tag}_factor.jsonl")):
    if l.startswith("{"):
        r = json.loads(l)
        fac[r["case"].strip()] = r
c3, c5, c4 = fac.get("C3"), fac.get("C5 s=0"), fac.get("C4")
par = [json.loads(l) for l in open(os.path.join(P, f"{tag}_parity.jsonl")) if l.startswith("{")]
okc = sorted({r["config"] for r in par if r.get("ok") and not r.get("partial") and not r.get("switches")})
part = [r for r in par if r.get("partial")]
rf = b["roofline"]
rows = [
    ("C2 GEMM 4096³ (bench `value`)", f"{b['ms_per_step']:.1f} ms", f"**{b['value']:.0f}** (1244)"),
    ("C2 end to end (pinned host buffers, H2D + D2H inside the timed region)",
     f"{2 * 4096 ** 3 / b['e2e']['value'] / 1e6:.1f} ms", f"{b['e2e']['value']:.0f} (1209)"),
    ("C4 LU n = 16384, nb = 256, lookahead", f"{c4['ms']:.0f} ms", f"**{c4['gflops']:.0f}** (1200)"),
    ("C5 LU n = 8192, s = 0", f"{c5['ms']:.1f} ms", f"**{c5['gflops']:.0f}** (1071)"),
    ("C3 Cholesky n = 8192, nb = 256, lookahead", f"{c3['ms']:.1f} ms", f"**{c3['gflops']:.0f}** (1043)"),
    ("CPU oracle, C2 sample on %d host cores (the reference arm)" % b["cpu_baseline"]["cores"], "—",
     f"{b['cpu_baseline']['value']:.2f}"),
]
tab = ["| Config | Time | Posit Gflop/s, round 2 (round 1) |", "|---|---|---|"] + [f"| {a} | {t} | {g} |" for a, t, g in rows]
note = (f"\n`profiles/{tag}_*`: CUDA events, median of 3 (C3, C5) / 2 (C4) runs after a warm-up, bench 10 steps; SM clock "
        f"{b['clocks']['sm_mhz']:.0f} MHz (max {b['clocks']['sm_max_mhz']:.0f}), throttle reasons {b['clocks']['reasons']}. "
        f"GEMM kernel: {rf['inst_per_mac']:.1f} instructions per MAC (ncu), **{rf['frac']:.2f} of the issue limit**, "
        f"FP64 pipe {rf.get('fp64_pipe', {}).get('frac', 0):.2f} busy. Every output word equal to the oracle's: "
        f"{', '.join(okc)}"
        + (f"; C4: rows 0..{part[0]['rows_compared'] - 1} (all columns) and ipiv's head" if part else "") + ".")
block = "\n".join(tab) + "\n" + note + "\n"
for f in ("README.md", "DESIGN.md"):
    p = os.path.join(ROOT, f)
    s = open(p).read()
    s2, n = re.subn(r"(<!-- R2_TABLE_BEGIN -->\n).*?(<!-- R2_TABLE_END -->)", lambda m: m.group(1) + block + m.group(2), s, flags=re.S)
    assert n == 1, f
    open(p, "w").write(s2)
print(block)
