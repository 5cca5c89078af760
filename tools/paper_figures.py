"""B200 analogs of the paper's GEMM figures (context measurements, not parity):

  Fig gemm_v100: GEMM Gflop/s vs operand scale sigma, N = 4096
  Fig gemm_gpu_all: GEMM Gflop/s vs N (sigma = 1)
  Fig gemm_trailing: trailing update N x K . K x N vs K, relative
                                 to the square GEMM rate

    python tools/paper_figures.py [--out profiles/paper_figures.jsonl]
Inputs: N(0, sigma^2) binary64 from numpy PCG64 (seeded), rounded to posit32
by posit_from_f64; C -= A B with the production posit_gemm; CUDA events.
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


def mk(shape, sigma, seed):
    return PB.posit_from_f64(torch.from_numpy(SI.normal_matrix(shape, sigma, seed)).cuda())


def time_gemm(A, B, C0, reps=3):
    C = C0.clone()
    PB.posit_gemm(A, B, C)
    ts = []
    for _ in range(reps):
        C.copy_(C0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        PB.posit_gemm(A, B, C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "paper_figures.jsonl"))
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    out = open(args.out, "w")

    def emit(r):
        print(json.dumps(r), flush=True)
        out.write(json.dumps(r) + "\n")
        out.flush()

    n = 4096
    for sigma in (1e-2, 1.0, 1e2, 1e4, 1e6):
        A, B, C = mk((n, n), sigma, 1), mk((n, n), sigma, 2), mk((n, n), sigma, 3)
        t = time_gemm(A, B, C)
        emit({"figure": "gemm_v100 analog (sigma sweep)", "N": n, "sigma": sigma, "gflops": 2 * n ** 3 / t / 1e9,
              "paper_v100_gflops": {1.0: 55, 1e6: 37}.get(sigma)})   # P:383-385 (sigma = 1 and 1e6 only)
    for n in (1024, 2048, 4096, 6144, 8192):
        A, B, C = mk((n, n), 1.0, 1), mk((n, n), 1.0, 2), mk((n, n), 1.0, 3)
        t = time_gemm(A, B, C, reps=2)
        emit({"figure": "gemm_gpu_all analog (N sweep)", "N": n, "sigma": 1.0, "gflops": 2 * n ** 3 / t / 1e9})
    square = None
    n = 16384
    for k in (1024, 512, 256, 128, 64, 32):
        A, B, C = mk((n, k), 1.0, 4), mk((k, n), 1.0, 5), mk((n, n), 1.0, 6)
        t = time_gemm(A, B, C, reps=2)
        g = 2.0 * n * n * k / t / 1e9
        square = square or g
        emit({"figure": "gemm_trailing analog (K sweep)", "N": n, "K": k, "gflops": g,
              "relative_to_K1024": g / square})
        del A, B, C
    out.close()


if __name__ == "__main__":
    main()
