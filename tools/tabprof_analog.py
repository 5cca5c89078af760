"""Tables tabrandom / tabprof analog: posit add by
operand range I0..I4 with the product's branch-free kernel (posit_vec_op) and
a SoftPosit-style loop kernel (tools/softposit_style.cu, the paper's decode /
encode loops), bits checked equal, ns per op per core and Gop/s.

    python tools/tabprof_analog.py [--count N] [--out profiles/tabprof_analog.jsonl]
    ncu --metrics smsp__inst_executed.sum,smsp__sass_average_branch_targets_threads_uniform.pct \
        python tools/tabprof_analog.py --count 1048576 --once     # instructions per op
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

CTRL_SRC = os.path.join(ROOT, "tools", "softposit_style.cu")
CTRL_LIB = os.path.join(ROOT, "tools", "libsoftposit_style.so")
PAPER_V100_ADD_NS = {"I0": 101, "I1": 215, "I2": 210, "I3": 148, "I4": 145}
PAPER_V100_ADD_NINST = {"I0": 81, "I1": 283, "I2": 237, "I3": 175, "I4": 150}


def ctrl():
    if not os.path.exists(CTRL_LIB) or os.path.getmtime(CTRL_LIB) < os.path.getmtime(CTRL_SRC):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-Xcompiler",
                        "-fPIC", "-shared", "-o", CTRL_LIB, CTRL_SRC], check=True)
    L = ctypes.CDLL(CTRL_LIB)
    L.softposit_style_add.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p]
    return L


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1 << 24)
    ap.add_argument("--once", action="store_true", help="one launch of each kernel per range (for ncu)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "tabprof_analog.jsonl"))
    args = ap.parse_args()
    L = ctrl()
    cores = torch.cuda.get_device_properties(0).multi_processor_count * 128
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    for lab in ("I0", "I1", "I2", "I3", "I4"):
        a = PB.posit_from_f64(torch.from_numpy(SI.range_samples(lab, args.count, seed=1)).cuda())
        b = PB.posit_from_f64(torch.from_numpy(SI.range_samples(lab, args.count, seed=2)).cuda())
        o1, o2 = torch.empty_like(a), torch.empty_like(a)
        ours = lambda: PB.posit_vec_op("add", a, b, o1)                                    # noqa: E731
        loop = lambda: L.softposit_style_add(a.data_ptr(), b.data_ptr(), o2.data_ptr(), a.numel(), st)  # noqa: E731
        if args.once:
            ours()
            loop()
            torch.cuda.synchronize()
            continue
        ours()
        loop()
        same = bool(torch.equal(o1, o2))
        t1, t2 = timed(ours), timed(loop)
        r = {"range": lab, "count": args.count, "bits_equal": same,
             "branch_free_ns_per_op_per_core": t1 * cores / args.count * 1e9,
             "loop_ns_per_op_per_core": t2 * cores / args.count * 1e9,
             "branch_free_gops": args.count / t1 / 1e9, "loop_gops": args.count / t2 / 1e9,
             "paper_v100_ns": PAPER_V100_ADD_NS[lab], "paper_v100_ninst": PAPER_V100_ADD_NINST[lab]}
        rows.append(r)
        print(json.dumps(r), flush=True)
    if rows:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
