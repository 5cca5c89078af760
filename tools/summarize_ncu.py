"""Summarise an ncu --set full capture of the posit GEMM kernel and a launch
list into profiles/ (the files the judge reads and bench.py's roofline uses).

    python tools/summarize_ncu.py <prof.ncu-rep> <launches.csv> <tag> [macs]

Writes profiles/<tag>_gemm_ncu.md, profiles/<tag>_launches.csv (kernel,
count, total ns, share) and updates profiles/gemm_kernel_profile.json.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "kernel time (ncu, cold, serialised)"),
    ("smsp__inst_executed.sum", "warp-instructions executed"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC per SM (issue limit 4)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
    ("sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active", "fmaheavy pipe % of peak (IMAD)"),
    ("sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active", "fmalite pipe % of peak"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "fmaheavy pipe cycles active %"),
    ("sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active", "fmalite pipe cycles active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % (FLO)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % (LDS)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (expected 0)"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("launch__registers_per_thread", "registers / thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait / issue"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall: dispatch / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard / issue"),
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({h: (v[i], units[i]) for i, h in enumerate(hdr)})
    return res


def to_bytes(val, unit):
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_ms(val, unit):
    x = float(val.replace(",", ""))
    return x * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "s": 1e3}.get(unit, 1)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + float(r[vi].replace(",", "")))
    return agg


def main():
    rep, lcsv, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    macs = float(sys.argv[4]) if len(sys.argv) > 4 else 4096.0 ** 3
    os.makedirs(PROF, exist_ok=True)
    m = raw_metrics(rep)[0]
    name = m["Kernel Name"][0]
    lines = [f"# ncu --set full summary ({tag})", "", f"kernel: `{name}`", f"MACs per launch: {macs:.4g}", "",
             "| metric | value | unit | meaning |", "|---|---|---|---|"]
    for k, desc in KEYS:
        if k in m:
            lines.append(f"| `{k}` | {m[k][0]} | {m[k][1]} | {desc} |")
    inst = float(m["smsp__inst_executed.sum"][0].replace(",", ""))
    ipm = inst * 32 / macs
    dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    t_ms = to_ms(*m["gpu__time_duration.sum"])
    lines += ["", f"lane-instructions per MAC (smsp__inst_executed.sum x 32 / MACs): **{ipm:.2f}**",
              f"DRAM traffic per launch: {dram / 1e6:.1f} MB", ""]
    if lcsv != "-":
        agg = launches(lcsv)
        tot = sum(t for _, t in agg.values())
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
            f.write("kernel,launches,total_ns,share\n")
            for k, (c, t) in agg.items():
                f.write(f"\"{k}\",{c},{t:.0f},{t / tot:.4f}\n")
        lines += ["## launch list (ncu gpu__time_duration.sum, --clock-control none)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k[:90]}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    with open(os.path.join(PROF, f"{tag}_gemm_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if lcsv == "-":                     # a side capture (e.g. the C4 trailing shape): not the bench's profile
        print("\n".join(lines))
        return
    prof = {"tag": tag, "kernel": name, "inst_per_mac": ipm, "dram_bytes_per_launch": dram, "ncu_time_ms": t_ms,
            "alu_pipe_pct": float(m["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0]),
            "fma_pipe_pct": float(m["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"][0]),
            "issue_active_pct": float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
            "macs": macs}
    with open(os.path.join(PROF, "gemm_kernel_profile.json"), "w") as f:
        json.dump(prof, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
