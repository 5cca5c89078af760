"""Copy one GPU session's evidence (gpurun_out/<dir>, written by tools/gpu_queue/evidence.sh)
into profiles/<tag>_* and print the results table for DESIGN.md / README.md.

    python tools/evidence_to_profiles.py gpurun_out/r2q3 r2q3
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
src, tag = sys.argv[1], sys.argv[2]


def rd(name):
    p = os.path.join(src, name)
    return open(p).read() if os.path.exists(p) else ""


def jl(text):
    return [json.loads(l) for l in text.splitlines() if l.startswith("{")]


def wr(name, text):
    if text:
        with open(os.path.join(PROF, f"{tag}_{name}"), "w") as f:
            f.write(text)


bench = jl(rd("bench.log"))
wr("bench.json", "\n".join(json.dumps(b) for b in bench) + "\n" if bench else "")
wr("factor.jsonl", "\n".join(l for l in rd("factor.log").splitlines() if l.startswith("{")) + "\n")
for n in ("chol_breakdown", "lu_breakdown", "lu_breakdown_c4"):
    wr(n + ".json", "\n".join(l for l in rd(n + ".log").splitlines() if l.startswith("{")) + "\n")
wr("parity.jsonl", rd("parity.jsonl") + rd("parity_serial.jsonl") + rd("parity_c4.jsonl"))
wr("pytest_gpu.txt", "\n".join(rd("pytest_gpu.log").splitlines()[-6:]) + "\n")
wr("smoke.txt", rd("smoke.log"))
wr("determinism.txt", rd("determinism.log"))
wr("env.txt", rd("env.txt"))
for n in ("launches.csv", "launches_chol.csv", "launches_lu.csv"):
    wr(n, rd(n))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


KEYS = ["launch__grid_size", "launch__block_size", "launch__cluster_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum"]
md = [f"# {tag}: ncu --set full --clock-control none (one launch each, inside the factorisation named)", ""]
for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
    m = raw(os.path.join(src, rep))
    if not m:
        continue
    md += [f"## `{rep}`: `{m['Kernel Name'][0][:110]}`", "", "| metric | value | unit |", "|---|---|---|"]
    md += [f"| `{k}` | {m[k][0]} | {m[k][1]} |" for k in KEYS if k in m]
    st = sorted(((float(v[0]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                 for k, v in m.items() if "issue_stalled" in k and k.endswith("_per_issue_active.ratio")
                 and "not_issued" not in k), reverse=True)
    md += ["", "stalls per issue: " + ", ".join(f"{n} {x:.2f}" for x, n in st[:6]), ""]
wr("ncu.md", "\n".join(md) + "\n")

if bench:
    b = bench[0]
    print(f"C2 GEMM: {b['value']:.0f} Gflop/s ({b['ms_per_step']:.2f} ms), e2e {b['e2e']['value']:.0f}, roofline frac "
          f"{b['roofline']['frac']:.3f} (inst/MAC {b['roofline']['inst_per_mac']:.2f}, stale {b['roofline']['inst_per_mac_stale']}), "
          f"parity {b['parity']['mismatches']}, clocks {b['clocks']}")
    for k in ("lu_c4", "chol_c3"):
        if k in b:
            print(f"{k}: {b[k]['value']:.0f} Gflop/s ({b[k]['ms_per_step']:.2f} ms) parity {b[k]['parity'].get('mismatches')} "
                  f"{b[k]['parity'].get('note', '')}")
    print("cpu_baseline", b.get("cpu_baseline"))
for r in jl(rd("factor.log")):
    print(f"{r['case']}: {r['ms']:.2f} ms  {r['gflops']:.0f} Gflop/s")
for n in ("chol_breakdown", "lu_breakdown", "lu_breakdown_c4"):
    for r in jl(rd(n + ".log")):
        print(n, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items() if k != "note"})
for r in jl(rd("parity.jsonl") + rd("parity_serial.jsonl") + rd("parity_c4.jsonl")):
    print("parity", r.get("config"), r.get("switches"), "ok" if r.get("ok") else r.get("skipped", "MISMATCH"),
          r.get("words_compared"), "partial rows %s" % r.get("rows_compared") if r.get("partial") else "")
print(rd("pytest_gpu.log").splitlines()[-2:] if rd("pytest_gpu.log") else "no pytest log")
