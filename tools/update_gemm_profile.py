"""Update the d_mac block of profiles/gemm_kernel_profile.json (what bench.py's roofline reads)
from an `ncu --set full` capture of k_gemm_d on C2 (4096^3), binding it to the SASS hash of the
library in the tree.      python tools/update_gemm_profile.py gpurun_out/r2q2/prof_gemm_d.ncu-rep r2q2
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

rep, tag = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
m = {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def f(k):
    return float(m[k][0].replace(",", ""))


def mb(k):
    return f(k) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m[k][1]]


path = os.path.join(ROOT, "profiles", "gemm_kernel_profile.json")
p = json.load(open(path))
d = p["d_mac"]
assert "k_gemm_d" in m["Kernel Name"][0] and "64, 128" in m["Kernel Name"][0], m["Kernel Name"][0]
macs = 4096.0 ** 3
d.update({
    "tag": tag, "kernel": m["Kernel Name"][0], "inst_per_mac": f("smsp__inst_executed.sum") * 32 / macs,
    "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
    "ncu_time_ms": f("gpu__time_duration.sum") * {"ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(m["gpu__time_duration.sum"][1], 1),
    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_pct": f("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "smem_bank_conflicts_ld": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
    "sass_sha256": bench.kernel_sass_sha(d["kernel_mangled"]),
    "sass_note": f"{tag} ncu capture ({rep}); bench.py flags inst_per_mac_stale when the running library's SASS differs",
})
json.dump(p, open(path, "w"), indent=1)
print({k: d[k] for k in ("tag", "inst_per_mac", "ncu_time_ms", "issue_active_pct", "fp64_pipe_pct", "sass_sha256")})
