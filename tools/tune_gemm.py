"""Time the posit GEMM tile variants on the hot-path shapes (run under gpurun).

    python tools/tune_gemm.py            # all variants, one subprocess each
Each variant must reproduce variant 0's bits exactly (same order contract).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [("C2 4096^3", 4096, 4096, 4096, "N"), ("LU trailing 16128x16128x256", 16128, 16128, 256, "N"),
          ("LU TRSM update 224x16128x32", 224, 16128, 32, "N"), ("SYRK-like NT 7936x7936x256", 7936, 7936, 256, "T"),
          ("SYRK lower 7936x7936x256", 7936, 7936, 256, "S"), ("SYRK lower 2048x2048x256", 2048, 2048, 256, "S"),
          ("Chol TRSM update NT 7936x224x32", 7936, 224, 32, "T"), ("Chol TRSM update NT 7936x32x32", 7936, 32, 32, "T"),
          ("panel update 16128x128x128", 16128, 128, 128, "N"), ("panel update 16256x32x32", 16256, 32, 32, "N")]

CHILD = r'''
import sys, json, hashlib, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2401_14117_b200 as PB
res = {}
for name, m, n, k, tb in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(1)
    def mk(r, c):
        return PB.posit_from_f64(torch.randn(r, c, generator=g, device="cuda", dtype=torch.float64))
    A = mk(m, k); B = mk(k, n) if tb == "N" else mk(n, k); C0 = mk(m, n); C = C0.clone()
    def run():
        if tb == "S":
            PB.posit_syrk(A, C)
        else:
            PB.posit_gemm(A, B, C, transb=tb)
    run()
    torch.cuda.synchronize()
    h = hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16]
    ts = []
    for _ in range(3):
        C.copy_(C0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[1]
    fl = (m * (m + 1) if tb == "S" else 2.0 * m * n) * k
    res[name] = {"ms": t, "gflops": fl/t/1e6, "sha": h}
print(json.dumps(res))
'''


def main():
    variants = [int(v) for v in sys.argv[1:]] or [0, 11, 12, 13, 14]
    out = {}
    for v in variants:
        env = dict(os.environ, POSIT_GEMM_VARIANT=str(v))
        code = f"ROOT={ROOT!r}\nSHAPES={SHAPES!r}\n" + CHILD
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            out[v] = {"error": r.stderr[-2000:]}
        else:
            out[v] = json.loads(r.stdout.strip().splitlines()[-1])
        print(json.dumps({"variant": v, **out[v]}), flush=True)
    ref = out.get(variants[0], {})
    for v in variants[1:]:
        for name in ref:
            if isinstance(ref.get(name), dict) and name in out.get(v, {}):
                assert out[v][name]["sha"] == ref[name]["sha"], (v, name, "bits differ between variants")
    print("all variants bit-identical", flush=True)


if __name__ == "__main__":
    main()
