#!/usr/bin/env python
"""Benchmark of the Posit(32,2) hot path on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload gemm|lu|cholesky]
                    [--impl ours|reference] [--force-dist] [--no-factor-keys]

Default workload = BASELINE.json configs[1], the metric's headline config:
Posit(32,2) GEMM C <- C - A.B, m = n = k = 4096, A, B, C ~ N(0,1) binary64 from
seed 1 rounded to posit32 (row-major uint32 patterns), every multiply and add
correctly rounded, ascending-k order.  A "step" is one such GEMM on fresh C
(C is restored from a resident copy inside the step: 64 MiB device copy).
At N = 1 it is the single-GPU C ABI call.  Under torchrun (N > 1, or with
--force-dist at N = 1) it is ONE 4096^3 problem split by column slabs of B and
C over the ranks, A broadcast from rank 0 over NCCL inside every step
(strong scaling).  value = 2 m n k / max-over-ranks step time.

Every run also carries the metric's other two rows at the same N:
  lu_c4    configs[3]: LU n = 16384, nb = 256 (2n^3/3 flops; getrf_dist over
           NCCL when distributed, else posit_getrf)
  chol_c3  configs[2]: Cholesky n = 8192, nb = 256 (n^3/3; potrf_dist / posit_potrf)
each with its own clocks and launches, and every output word of C2, C4 and C3
compared with the committed oracle digests (tests/golden/config_digests,
written by tools/oracle_digests.py): "parity" keys.

--workload lu|cholesky  make configs[3] / configs[2] the main line
--impl reference        the CPU oracle (oracle/), on this box's host cores, on a
                        bounded sample of the same workload (rank 0 only).

Extra keys: roofline (issue-slot roofline of the GEMM kernel and its FP64-pipe use,
instruction count bound to the kernel's SASS hash), cpu_baseline (oracle
sample), e2e (posit_gemm_host with pinned host buffers, copies inside the timed
region), clocks (nvidia-smi during the timed region), gpu_launches (our kernel
launches in the timed region).
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
            "scaling": "strong" if args.gpus > 1 or args.workload != "gemm" else "weak", "vs_baseline": None,
            "dtype": "posit32 (CPU oracle: integer arithmetic)", "data": "synthetic",
            "config": _config(args, args.gpus, args.gpus > 1), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "Gflop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config(args, world=1, dist_on=False):
    if args.workload == "gemm":
        return {"workload": "configs[1]: Posit(32,2) GEMM C -= A.B, m=n=k=4096, N(0,1) seed 1, row-major",
                "m": 4096, "n": 4096, "k": 4096, "order": "ascending-k, per-op RNE, no quire",
                "l2": "inputs (3 x 64 MiB) larger than the 126 MB L2",
                "parallelism": (f"C split by column slabs over {world} rank(s), A broadcast over NCCL each step "
                                "(one problem, strong scaling)" if dist_on else "single GPU")}
    if args.workload == "lu":
        return {"workload": "configs[3]: Posit(32,2) LU with partial pivoting, n=16384, nb=256, U[-1,1) seed 3",
                "n": 16384, "nb": 256, "l2": "matrix 1 GiB > L2",
                "parallelism": (f"1x{world} column-block-cyclic, NCCL panel broadcast" if dist_on else "single GPU")}
    return {"workload": "configs[2]: Posit(32,2) Cholesky, n=8192, nb=256, A = G G^T/n + I seed 2",
            "n": 8192, "nb": 256, "l2": "matrix 256 MiB > L2",
            "parallelism": (f"1x{world} column-block-cyclic, NCCL panel broadcast" if dist_on else "single GPU")}


# ---------------------------------------------------------------------- our arm
DIGESTS = os.path.join(ROOT, "tests", "golden", "config_digests")


def parity_vs_oracle(cfg, M, ipiv=None, info=None):
    """Every output word of this run against the committed oracle digests
    (tests/golden/config_digests/<cfg>.json, written by tools/oracle_digests.py
    from the CPU oracle alone): per-row SHA-256 + whole-output SHA-256."""
    import hashlib
    ref = _load_json(os.path.join(DIGESTS, f"{cfg}.json"))
    M = np.ascontiguousarray(M).view(np.uint32)
    h = hashlib.sha256(M.tobytes())
    if ipiv is not None:
        h.update(np.ascontiguousarray(ipiv, np.int32).tobytes())
    if info is not None:
        h.update(np.array([info], np.int32).tobytes())
    out = {"config": cfg, "words": int(M.size), "gpu_sha": h.hexdigest()}
    if ref is None:
        # an LU oracle run that stopped at a checkpoint after k steps: rows < k and ipiv[:k] are final
        part = _load_json(os.path.join(DIGESTS, f"{cfg}_partial.json"))
        if part is None:
            out.update({"oracle_sha": None, "mismatches": None, "note": "no oracle digest committed for this config"})
            return out
        k = int(part["partial_rows"])
        rows = [hashlib.sha256(M[i].tobytes()).hexdigest()[:16] for i in range(k)]
        bad = [i for i, (g, o) in enumerate(zip(rows, part["row_digests"])) if g != o]
        ip_ok = ipiv is not None and hashlib.sha256(
            np.ascontiguousarray(ipiv[:k], np.int32).tobytes()).hexdigest() == part["ipiv_head_sha256"]
        out.update({"oracle_sha": None, "partial_rows": k, "words_compared": int(k * M.shape[1]),
                    "mismatched_rows": len(bad), "first_bad_row": bad[0] if bad else None, "ipiv_head_match": ip_ok,
                    "mismatches": 0 if (not bad and ip_ok) else max(1, len(bad)),
                    "note": f"oracle run checkpointed after {k} of {part['of_rows']} steps: rows < {k} "
                            f"(all columns) and ipiv[:{k}] are final and compared; the rest is not",
                    "oracle_version": part["oracle_sha256"][:16]})
        return out
    rows = [hashlib.sha256(M[i].tobytes()).hexdigest()[:16] for i in range(M.shape[0])]
    bad = [i for i, (g, o) in enumerate(zip(rows, ref["row_digests"])) if g != o]
    out.update({"oracle_sha": ref["output_sha256"], "mismatched_rows": len(bad),
                "first_bad_row": bad[0] if bad else None,
                "mismatches": 0 if (not bad and out["gpu_sha"] == ref["output_sha256"]) else max(1, len(bad)),
                "oracle_version": ref["oracle_sha256"][:16]})
    return out


def _timed(step, steps, warmup, stream, barrier, local, dist_on, PB):
    """W untimed steps; K steps between barrier + synchronize, CUDA events on
    the launching stream, nvidia-smi clocks during the timed region; returns
    (max-over-ranks ms per step, clocks, our kernel launches)."""
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        launches0 = PB.posit_kernel_launches()
        ev0.record(stream)
        for _ in range(steps):
            step()
        ev1.record(stream)
        launches = PB.posit_kernel_launches() - launches0
        barrier()
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=torch.device("cuda", local))
    if dist_on:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / steps, clk.summary(), launches


def _gather_cols(local, desc, world):
    """Full matrix from every rank's column blocks (rank 0 result; outside timing)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return desc.gather([local]) if desc is not None else local
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous())
    return desc.gather(parts)


def factor_key(kind, args, dev, stream, barrier, local, rank, world, dist_on, PB):
    """lu_c4 (configs[3], n = 16384, nb = 256) or chol_c3 (configs[2], n = 8192,
    nb = 256): the factorisation on all ranks (1 x P column-block-cyclic over
    NCCL when distributed, else the single-GPU C ABI), timed like the main line,
    with its own clocks and a word-by-word parity check of the factors."""
    import torch
    import synthetic_inputs as SI
    from paper_2401_14117_b200.dist import BlockCyclic1D, getrf_dist, potrf_dist
    lu = kind == "lu"
    nn, nb = (SI.C4_N, SI.C4_NB) if lu else (SI.C3_N, SI.C3_NB)
    full = PB.posit_from_f64(torch.from_numpy(SI.config4() if lu else SI.config3()).to(dev))
    ipiv = torch.zeros(nn, dtype=torch.int32, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    desc = BlockCyclic1D(nn, nb, world, rank) if dist_on else None
    dA0 = desc.scatter(full) if dist_on else full
    del full
    dA = dA0.clone()
    if lu:
        def step():
            dA.copy_(dA0)
            if dist_on:
                getrf_dist(dA, desc, ipiv, info)
            else:
                PB.posit_getrf(dA, ipiv, info, nb=nb)
    else:
        def step():
            dA.copy_(dA0)
            if dist_on:
                potrf_dist(dA, desc, info)
            else:
                PB.posit_potrf(dA, info, nb=nb)
    steps, warmup = (args.factor_steps, 1) if lu else (max(3, args.factor_steps), 3)
    ms, clocks, launches = _timed(step, steps, warmup, stream, barrier, local, dist_on, PB)
    flops = 2.0 * nn ** 3 / 3 if lu else nn ** 3 / 3.0
    M = _gather_cols(dA, desc, world)
    out = None
    if rank == 0:
        cfg = "C4" if lu else "C3"
        out = {"workload": ("configs[3]: LU with partial pivoting n=16384 nb=256 U[-1,1) seed 3" if lu else
                            "configs[2]: Cholesky n=8192 nb=256 A = G G^T/n + I seed 2"),
               "value": flops / (ms * 1e-3) / 1e9, "unit": "Gflop/s", "ms_per_step": ms, "steps": steps,
               "warmup": warmup, "flops": flops,
               "parallelism": (f"1x{world} column-block-cyclic, NCCL panel broadcast, lookahead" if dist_on
                               else "single GPU (posit_getrf / posit_potrf, lookahead)"),
               "scaling": "strong", "clocks": clocks, "gpu_launches": launches,
               "info": int(info.cpu()[0]),
               "parity": parity_vs_oracle(cfg, M.cpu().numpy(), ipiv.cpu().numpy() if lu else None,
                                          int(info.cpu()[0]))}
    del dA, dA0, M
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2401_14117_b200 as PB
    import synthetic_inputs as SI
    from paper_2401_14117_b200.dist import col_slab, gemm_colsplit

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dist_on = world > 1 or args.force_dist
    if dist_on:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    def barrier():
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    line = None
    if args.workload == "gemm":
        # ---- configs[1]: inputs resident in HBM (converted by our posit_from_f64 kernel)
        m = n = k = 4096
        A64, B64, C64 = SI.config2()
        c0, c1 = col_slab(n, world, rank) if dist_on else (0, n)
        dA = PB.posit_from_f64(torch.from_numpy(A64).to(dev))
        dB = PB.posit_from_f64(torch.from_numpy(np.ascontiguousarray(B64[:, c0:c1])).to(dev))
        dC0 = PB.posit_from_f64(torch.from_numpy(np.ascontiguousarray(C64[:, c0:c1])).to(dev))
        del A64, B64, C64
        if dist_on and rank != 0:
            dA.zero_()                      # only rank 0 holds A; the step broadcasts it
        dC = dC0.clone()
        flops = 2.0 * m * n * k             # ONE problem over all ranks (strong scaling when distributed)

        def step():
            dC.copy_(dC0)
            if dist_on:
                gemm_colsplit(dA, dB, dC, src=0)
            else:
                PB.posit_gemm(dA, dB, dC)
        ms_per_step, clocks, launches = _timed(step, args.steps, args.warmup, stream, barrier, local, dist_on, PB)
        value = flops / (ms_per_step * 1e-3) / 1e9
        Cfull = _gather_cols_slabs(dC, world, n) if dist_on else dC
        if rank == 0:
            line = {"metric": METRIC, "value": value, "unit": "Gflop/s", "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                    "scaling": "strong" if dist_on else "weak",
                    "vs_baseline": None, "dtype": _dtype(),
                    "data": "synthetic (seeded numpy PCG64, BASELINE recipe)", "config": _config(args, world, dist_on),
                    "clocks": clocks, "gpu_launches": launches,
                    "parity": parity_vs_oracle("C2", Cfull.cpu().numpy()),
                    "paper_context": {"gemm_gflops_rtx4090_n8000": 181.4, "gemm_gflops_agilex_n8000": 202.7,
                                      "lu_gflops_rx7900_n8000": 13.4, "source": "PAPER.md:403,432,542"}}
            pw = clocks.get("power_w_median")
            line["efficiency"] = {"board_power_w": pw, "gflops_per_w": (value / world / pw) if pw else None,
                                  "paper": "LU 0.076 Gflops/W RX7900 + host, AC wall (P:591)"}
            # ---- roofline of the dominant kernel (this rank's GEMM), timed alone on this stream
            line["roofline"] = gemm_roofline(PB, dA, dB, dC, dC0, m, c1 - c0, k, stream)
        del Cfull
        # ---- end to end through the C ABI with HOST buffers (this rank's slab)
        hA = torch.from_numpy(dA.cpu().numpy()).pin_memory()
        hB = torch.from_numpy(dB.cpu().numpy()).pin_memory()
        hC0 = dC0.cpu()
        hC = hC0.clone().pin_memory()
        work = torch.empty(PB.posit_gemm_host_work_bytes(m, c1 - c0, k), dtype=torch.uint8, device=dev)
        for _ in range(2):
            hC.copy_(hC0)
            PB.posit_gemm_host(hA, hB, hC, work)
        e2e_steps = max(2, min(args.steps, 5))
        # one pinned input copy of C per timed step, made before the timed region (the call
        # overwrites C in place; re-filling it on the host is not part of the API call)
        hCs = [hC0.clone().pin_memory() for _ in range(e2e_steps)]
        barrier()
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            PB.posit_gemm_host(hA, hB, hCs[i], work)
        torch.cuda.synchronize()
        e2e = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=dev)
        if dist_on:
            dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
        if rank == 0:
            line["e2e"] = {"value": flops / float(e2e.item()) / 1e9, "unit": "Gflop/s",
                           "h2d_bytes_per_step": world * (m * k + k * (c1 - c0)) * 4 if dist_on else 3 * m * k * 4,
                           "d2h_bytes_per_step": m * n * 4,
                           "api": "posit_gemm_host per rank on its slab (pinned host A, B, C; "
                                  "H2D + kernel + D2H + sync per step)"}
            if dist_on:
                line["e2e"]["h2d_bytes_per_step"] = world * m * k * 4 + k * n * 4 + m * n * 4
            elif (m, n, k) == (4096, 4096, 4096):
                # the host buffer the first timed call wrote: every word against the oracle digests
                pe = parity_vs_oracle("C2", hCs[0].numpy())
                line["e2e"]["parity"] = {k_: pe.get(k_) for k_ in ("gpu_sha", "oracle_sha", "mismatched_rows",
                                                                    "mismatches")}
        del dA, dB, dC, dC0, work
        torch.cuda.empty_cache()
        # ---- LU (configs[3]) and Cholesky (configs[2]) at this N: the metric's other two rows
        if not args.no_factor_keys:
            for kind, key in (("lu", "lu_c4"), ("cholesky", "chol_c3")):
                r = factor_key(kind, args, dev, stream, barrier, local, rank, world, dist_on, PB)
                if rank == 0:
                    line[key] = r
    else:
        r = factor_key("lu" if args.workload == "lu" else "cholesky", args, dev, stream, barrier, local, rank,
                       world, dist_on, PB)
        if rank == 0:
            line = {"metric": METRIC, "value": r["value"], "unit": "Gflop/s", "n_gpus": world,
                    "steps": r["steps"], "warmup": r["warmup"], "ms_per_step": r["ms_per_step"],
                    "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                    "dtype": _dtype(),
                    "data": "synthetic (seeded numpy PCG64, BASELINE recipe)",
                    "config": _config(args, world, dist_on), "clocks": r["clocks"],
                    "gpu_launches": r["gpu_launches"], "parity": r["parity"]}

    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_sample(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _gather_cols_slabs(dC, world, n):
    """C (m x n) from the ranks' contiguous column slabs (col_slab)."""
    import torch
    import torch.distributed as dist
    from paper_2401_14117_b200.dist import col_slab
    m = dC.shape[0]
    q = col_slab(n, world, 0)[1]
    buf = torch.zeros((m, q), dtype=dC.dtype, device=dC.device)
    buf[:, : dC.shape[1]] = dC
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = torch.empty((m, n), dtype=dC.dtype, device=dC.device)
    for r in range(world):
        c0, c1 = col_slab(n, world, r)
        out[:, c0:c1] = parts[r][:, : c1 - c0]
    return out


def kernel_sass_sha(kernel_mangled: str):
    """SHA-256 of the SASS of one kernel of the loaded library (cuobjdump), so a
    stored ncu instruction count can be checked against the binary that runs."""
    import hashlib
    import re
    import paper_2401_14117_b200 as PB
    lib = PB.lib()._name
    exe = "cuobjdump"
    for cand in ("/usr/local/cuda/bin/cuobjdump",):
        if os.path.exists(cand):
            exe = cand
    try:
        txt = subprocess.run([exe, "-sass", "-fun", kernel_mangled, lib], capture_output=True, text=True,
                             timeout=120).stdout
    except Exception:
        return None
    body = [l.strip() for l in txt.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    return hashlib.sha256("\n".join(body).encode()).hexdigest() if body else None


def _dtype() -> str:
    mac = "integer-pipe MAC" if os.environ.get("POSIT_GEMM_PATH", "1") == "0" else "binary64-pipe MAC"
    return f"posit32 (every mul/add one correctly rounded Posit(32,2) op; {mac})"


def gemm_roofline(PB, dA, dB, dC, dC0, m, n, k, stream):
    """Issue-slot roofline of the GEMM kernel, timed live with CUDA events on the
    launching stream (copy excluded), against SMs x 128 lanes x clock (one
    warp-instruction per SMSP per clock).  Both MACs are bound by issue plus
    their busiest pipe: the integer MAC by the ALU pipe, the binary64-pipe MAC
    (the default) by the FP64 pipe, whose use is reported beside the issue
    fraction (its own measured rate, profiles/pipebench_b200.json)."""
    import torch
    peaks = _load_json(PEAKS_PATH) or {}
    allp = _load_json(PROFILE_PATH) or {}
    dpath = os.environ.get("POSIT_GEMM_PATH", "1") != "0"
    prof = allp.get("d_mac", {}) if dpath else allp
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
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
    src = f"ncu smsp__inst_executed.sum x 32 / MACs (profiles/gemm_kernel_profile.json, {prof.get('tag')})"
    if inst_per_mac is None:
        inst_per_mac = prof.get("static_inst_per_mac", 54.1)
        src = "static SASS count of the inner loop (tools/sass_loop.py); no ncu capture yet"
    sass = kernel_sass_sha(prof["kernel_mangled"]) if prof.get("kernel_mangled") else None
    peak = n_sm * LANES_PER_SM * f_max / 1e12
    achieved = macs * inst_per_mac / t / 1e12
    out = {"bound": "alu", "unit": "Tinst/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
           "traffic": prof.get("dram_bytes_per_launch"), "kernel": prof.get("kernel", "pg::k_gemm (NN)"),
           "kernel_ms": t * 1e3, "inst_per_mac": inst_per_mac, "inst_per_mac_source": src,
           "sass_sha256": sass, "inst_per_mac_stale": (None if sass is None else sass != prof.get("sass_sha256")),
           "peak_source": f"{n_sm} SMs x 4 SMSP x 32 lanes x sm_max_mhz {f_max / 1e6:.0f} (MEASURED_PEAKS.json) "
                          "= warp-instruction issue limit; see DESIGN.md",
           "posit_tflops_kernel": 2 * macs / t / 1e12,
           "mac": "binary64 pipe (D-MAC)" if dpath else "integer pipes"}
    if dpath and prof.get("fp64_cycles_per_mac"):
        # binary64 pipe: its busy cycles per warp-MAC (DADD / DMUL 1 / 1.83, DFMA 1 / 1.47 SM-clocks,
        # measured) against the clock
        busy = macs / 32.0 * prof["fp64_cycles_per_mac"] / n_sm / (t * f_max)
        out["fp64_pipe"] = {"frac": busy, "fp64_inst_per_mac": prof.get("fp64_inst_per_mac"),
                            "cycles_per_warp_mac": prof["fp64_cycles_per_mac"],
                            "source": "profiles/pipebench_b200.json rates x the kernel's FP64 instruction mix"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", choices=["gemm", "lu", "cholesky"], default="gemm")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the distributed (NCCL) schedules even at world size 1")
    ap.add_argument("--no-factor-keys", action="store_true", help="skip the lu_c4 / chol_c3 keys")
    ap.add_argument("--factor-steps", type=int, default=3, help="timed steps of the lu_c4 / chol_c3 keys")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
