"""Table tabrandom analog on B200 (NEXT-2): elementwise posit
Add / Mul / Div / Sqrt throughput by operand range I0..I4.

    python tools/op_microbench.py [--count 16777216] [--out profiles/op_microbench.jsonl]

Operands: log-uniform magnitudes from each range of Table tabrandom
(I0 = [1,2), I1 = [1e-38,1e-30), I2 = [1e30,1e38), I3 = [1e-15,1e-14),
I4 = [1e14,1e15); random signs), rounded to Posit(32,2).  Each op runs
posit_vec_op (the branch-free __clz decode of csrc/posit32.cuh) over
`count` pairs; time by CUDA events (median of 5, after warm-up).  Reported
as ns per op per CUDA core like the paper (time x cores / ops, cores = SMs x
128) and as Gop/s.  The paper's V100 SoftPosit port: 101 / 101 / 173 / 96 ns
on I0 and up to 215 / 209 / 309 / 148 on I1 (magnitude-dependent loops).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB  # noqa: E402
import synthetic_inputs as SI  # noqa: E402

PAPER_V100_NS = {"I0": (101, 101, 173, 96), "I1": (215, 209, 301, 143), "I2": (210, 209, 309, 148),
                 "I3": (148, 141, 233, 136), "I4": (145, 141, 230, 136)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1 << 24)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "op_microbench.jsonl"))
    args = ap.parse_args()
    props = torch.cuda.get_device_properties(0)
    cores = props.multi_processor_count * 128
    rows = []
    for lab in ("I0", "I1", "I2", "I3", "I4"):
        a = PB.posit_from_f64(torch.from_numpy(SI.range_samples(lab, args.count, seed=1)).cuda())
        b = PB.posit_from_f64(torch.from_numpy(SI.range_samples(lab, args.count, seed=2)).cuda())
        out = torch.empty_like(a)
        res = {"range": lab, "count": args.count, "cores": cores}
        for i, op in enumerate(("add", "mul", "div", "sqrt")):
            x = a.abs() if op == "sqrt" else a          # sqrt of |a| (abs of a pattern is exact)
            for _ in range(3):
                PB.posit_vec_op(op, x, b, out)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                PB.posit_vec_op(op, x, b, out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            t = float(np.median(ts))
            res[f"{op}_ns_per_op_per_core"] = t * cores / args.count * 1e9
            res[f"{op}_gops"] = args.count / t / 1e9
            res[f"{op}_paper_v100_ns"] = PAPER_V100_NS[lab][i]
        rows.append(res)
        print(json.dumps(res), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
