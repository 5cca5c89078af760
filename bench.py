#!/usr/bin/env python
"""Benchmark of the Posit(32,2) hot path on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload gemm|lu|cholesky]
                    [--impl ours|reference]

Default workload = BASELINE.json configs[1], the metric's headline config:
Posit(32,2) GEMM C <- C - A.B, m = n = k = 4096, A, B, C ~ N(0,1) binary64 from
seed 1 rounded to posit32 (row-major uint32 patterns), every multiply and add
correctly rounded, ascending-k order.  A "step" is one such GEMM on fresh C
(C is restored from a resident copy inside the step: 64 MiB device copy).
value = posit Gflop/s = 2 m n k / step time, summed over ranks (each rank runs
its own configs[1] problem: weak scaling, no data-path collective).

--workload lu        configs[3] at N=1 (n = 16384, nb = 256), 2n^3/3 flops
--workload cholesky  configs[2] (n = 8192, nb = 256), n^3/3 flops
--impl reference     the CPU oracle (oracle/), on this box's host cores, on a
                     bounded sample of the same workload (rank 0 only).

Extra keys: roofline (issue-bound integer ALU roofline of the GEMM kernel),
cpu_baseline (oracle sample), e2e (posit_gemm_host with pinned host buffers,
copies inside the timed region), clocks (nvidia-smi during the timed region),
gpu_launches (our kernel launches in the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Posit(32,2) Gflop/s (GEMM 2mnk; LU 2n^3/3; Cholesky n^3/3)"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_PATH = os.path.join(ROOT, "profiles", "gemm_kernel_profile.json")
N_SM = 148
LANES_PER_SM = 128        # 4 SMSPs x 1 warp-instruction (32 lanes) per clock: the issue limit


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                parts = [p.strip() for p in out.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": float(np.median(pw)) if pw else None}


def _load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------- reference arm
def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_oracle_sample(workload: str, target_s: float = 12.0):
    """Time the oracle (as it stands) on a bounded sample of the workload."""
    from oracle import oracle as O
    import synthetic_inputs as SI
    cores = O.num_threads()
    if workload == "gemm":
        A, B, C = SI.config2()
        Bp = O.from_f64_array(B)
        rows = 1
        while True:
            Ap, Cp = O.from_f64_array(A[:rows]), O.from_f64_array(C[:rows])
            t0 = time.perf_counter()
            O.gemm(Ap, Bp, Cp)
            dt = time.perf_counter() - t0
            if dt >= target_s or rows >= 4096:
                break
            rows = min(4096, max(rows * 2, int(rows * target_s / max(dt, 1e-3) * 1.1)))
        flops = 2.0 * rows * 4096 * 4096
        return {"value": flops / dt / 1e9, "unit": "Gflop/s", "cores": cores, "kind": "oracle",
                "sample": f"{rows} of 4096 output rows of configs[1] GEMM (full k=4096 chains), {dt:.1f} s",
                "seconds": dt, "cpu_model": _cpu_model()}
    # LU / Cholesky: the oracle's textbook loop on a leading n_s x n_s sample of the same recipe
    n_s = 256
    while True:
        if workload == "lu":
            Ap = O.from_f64_array(SI.lu_matrix(n_s, SI.C4_SEED))
            t0 = time.perf_counter()
            O.getrf(Ap)
            dt = time.perf_counter() - t0
            flops = 2.0 * n_s ** 3 / 3
        else:
            Ap = O.from_f64_array(SI.config3(n_s))
            t0 = time.perf_counter()
            O.potrf_lower(Ap)
            dt = time.perf_counter() - t0
            flops = n_s ** 3 / 3.0
        if dt >= target_s / 4 or n_s >= 2048:
            break
        n_s = int(n_s * 1.26 ** 3)   # ~2x work steps
    return {"value": flops / dt / 1e9, "unit": "Gflop/s", "cores": cores, "kind": "oracle",
            "sample": f"{workload} of the same recipe at n={n_s} (oracle textbook loop), {dt:.1f} s", "seconds": dt,
            "cpu_model": _cpu_model()}


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    res = []
    steps = max(1, args.steps)
    cb = None
    for i in range(args.warmup + steps):
        cb = cpu_oracle_sample(args.workload, target_s=4.0)
        if i >= args.warmup:
            res.append(cb["value"])
    v = float(np.median(res))
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Gflop/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": cb["seconds"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "posit32 (int32 ALU)", "data": "synthetic",
            "config": _config(args), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "Gflop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config(args):
    if args.workload == "gemm":
        return {"workload": "configs[1]: Posit(32,2) GEMM C -= A.B, m=n=k=4096, N(0,1) seed 1, row-major",
                "m": 4096, "n": 4096, "k": 4096, "order": "ascending-k, per-op RNE, no quire",
                "l2": "inputs (3 x 64 MiB) larger than the 126 MB L2", "parallelism": f"replica x{args.gpus}"}
    if args.workload == "lu":
        return {"workload": "configs[3] at 1 GPU: Posit(32,2) LU with partial pivoting, n=16384, nb=256, U[-1,1) seed 3",
                "n": 16384, "nb": 256, "l2": "matrix 1 GiB > L2",
                "parallelism": (f"1x{args.gpus} column-block-cyclic, NCCL panel broadcast" if args.gpus > 1 else "single GPU")}
    return {"workload": "configs[2]: Posit(32,2) Cholesky, n=8192, nb=256, A = G G^T/n + I seed 2",
            "n": 8192, "nb": 256, "l2": "matrix 256 MiB > L2",
            "parallelism": (f"1x{args.gpus} column-block-cyclic, NCCL panel broadcast" if args.gpus > 1 else "single GPU")}


# ---------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2401_14117_b200 as PB
    import synthetic_inputs as SI

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- inputs resident in HBM (converted by our posit_from_f64 kernel) ----
    if args.workload == "gemm":
        m = n = k = 4096
        A64, B64, C64 = SI.config2()
        dA = PB.posit_from_f64(torch.from_numpy(A64).to(dev))
        dB = PB.posit_from_f64(torch.from_numpy(B64).to(dev))
        dC0 = PB.posit_from_f64(torch.from_numpy(C64).to(dev))
        dC = dC0.clone()
        flops = 2.0 * m * n * k

        def step():
            dC.copy_(dC0)
            PB.posit_gemm(dA, dB, dC)
    elif args.workload == "lu":
        nn = SI.C4_N
        full = PB.posit_from_f64(torch.from_numpy(SI.config4()).to(dev))
        ipiv = torch.zeros(nn, dtype=torch.int32, device=dev)
        info = torch.zeros(1, dtype=torch.int32, device=dev)
        flops = 2.0 * nn ** 3 / 3
        if world > 1:
            # configs[3]: ONE n = 16384 LU shared by all ranks (1 x P column-block-cyclic, NCCL panel broadcast)
            from paper_2401_14117_b200.dist import BlockCyclic1D, getrf_dist
            desc = BlockCyclic1D(nn, SI.C4_NB, world, rank)
            dA0 = desc.scatter(full)
            del full
            dA = dA0.clone()

            def step():
                dA.copy_(dA0)
                getrf_dist(dA, desc, ipiv, info)
        else:
            dA0 = full
            dA = dA0.clone()

            def step():
                dA.copy_(dA0)
                PB.posit_getrf(dA, ipiv, info, nb=SI.C4_NB)
    else:
        nn = SI.C3_N
        full = PB.posit_from_f64(torch.from_numpy(SI.config3()).to(dev))
        info = torch.zeros(1, dtype=torch.int32, device=dev)
        flops = nn ** 3 / 3.0
        if world > 1:
            # configs[2]: ONE n = 8192 Cholesky shared by all ranks (1 x P column-block-cyclic)
            from paper_2401_14117_b200.dist import BlockCyclic1D, potrf_dist
            desc = BlockCyclic1D(nn, SI.C3_NB, world, rank)
            dA0 = desc.scatter(full)
            del full
            dA = dA0.clone()

            def step():
                dA.copy_(dA0)
                potrf_dist(dA, desc, info)
        else:
            dA0 = full
            dA = dA0.clone()

            def step():
                dA.copy_(dA0)
                PB.posit_potrf(dA, info, nb=SI.C3_NB)
    # whole-job work: the GEMM runs one problem per rank (weak scaling); LU and
    # Cholesky are one problem distributed over all ranks (strong scaling)
    strong = args.workload in ("lu", "cholesky") and world > 1
    job_flops = flops if strong else world * flops

    for _ in range(args.warmup):
        step()
    barrier()

    # ---- timed region -------------------------------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        launches0 = PB.posit_kernel_launches()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        launches = PB.posit_kernel_launches() - launches0
        barrier()
    t_ms = ev0.elapsed_time(ev1)
    t_tensor = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    t_max = float(t_tensor.item())
    ms_per_step = t_max / args.steps
    value = job_flops / (ms_per_step * 1e-3) / 1e9

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gflop/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "posit32 (int32 ALU; every mul/add correctly rounded)",
                "data": "synthetic (seeded numpy PCG64, BASELINE recipe)", "config": _config(args),
                "clocks": clk.summary(), "gpu_launches": launches,
                "paper_context": {"gemm_gflops_rtx4090_n8000": 181.4, "gemm_gflops_agilex_n8000": 202.7,
                                  "lu_gflops_rx7900_n8000": 13.4, "source": "PAPER.md:403,432,542"}}

    # ---- energy efficiency (Table PowerE analog): NVML board power of
    # this GPU during the timed region, not the paper's AC wall power
    if rank == 0:
        pw = line["clocks"].get("power_w_median")
        line["efficiency"] = {"board_power_w": pw, "gflops_per_w": (value / world / pw) if pw else None,
                              "paper": "LU 0.076 Gflops/W RX7900 + host, AC wall (P:591)"}

    # ---- roofline of the dominant kernel (GEMM), timed alone on this stream --
    if args.workload == "gemm" and rank == 0:
        line["roofline"] = gemm_roofline(PB, dA, dB, dC, dC0, m, n, k, stream)

    # ---- end to end through the C ABI with HOST buffers ----------------------
    if args.workload == "gemm":
        hA = torch.from_numpy(dA.cpu().numpy()).pin_memory()
        hB = torch.from_numpy(dB.cpu().numpy()).pin_memory()
        hC0 = dC0.cpu()
        hC = hC0.clone().pin_memory()
        work = torch.empty(PB.posit_gemm_host_work_bytes(m, n, k), dtype=torch.uint8, device=dev)
        for _ in range(2):
            hC.copy_(hC0)
            PB.posit_gemm_host(hA, hB, hC, work)
        barrier()
        e2e_steps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            hC.copy_(hC0)
            PB.posit_gemm_host(hA, hB, hC, work)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        e2e = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
        if rank == 0:
            line["e2e"] = {"value": world * flops / float(e2e.item()) / 1e9, "unit": "Gflop/s",
                           "h2d_bytes_per_step": 3 * m * k * 4, "d2h_bytes_per_step": m * n * 4,
                           "api": "posit_gemm_host (pinned host A, B, C; H2D + kernel + D2H + sync per step)"}

    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_sample(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def gemm_roofline(PB, dA, dB, dC, dC0, m, n, k, stream):
    """Issue-bound integer roofline of the GEMM kernel, timed live with CUDA events
    on the launching stream (copy excluded), against 148 SMs x 128 lanes x clock."""
    import torch
    peaks = _load_json(PEAKS_PATH) or {}
    prof = _load_json(PROFILE_PATH) or {}
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    times = []
    for _ in range(5):
        dC.copy_(dC0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        PB.posit_gemm(dA, dB, dC)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(times))
    macs = float(m) * n * k
    inst_per_mac = prof.get("inst_per_mac")
    src = "ncu smsp__inst_executed.sum x 32 / MACs (profiles/gemm_kernel_profile.json)"
    if inst_per_mac is None:
        inst_per_mac = prof.get("static_inst_per_mac", 54.1)
        src = "static SASS count of the inner loop (tools/sass_stats.py); no ncu capture yet"
    peak = N_SM * LANES_PER_SM * f_max / 1e12
    achieved = macs * inst_per_mac / t / 1e12
    return {"bound": "alu", "unit": "Tinst/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
            "traffic": prof.get("dram_bytes_per_launch"), "kernel": prof.get("kernel", "pg::k_gemm (NN)"),
            "kernel_ms": t * 1e3, "inst_per_mac": inst_per_mac, "inst_per_mac_source": src,
            "peak_source": f"148 SMs x 4 SMSP x 32 lanes x sm_max_mhz {f_max / 1e6:.0f} (MEASURED_PEAKS.json) "
                           "= warp-instruction issue limit; see DESIGN.md",
            "posit_tflops_kernel": 2 * macs / t / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", choices=["gemm", "lu", "cholesky"], default="gemm")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
