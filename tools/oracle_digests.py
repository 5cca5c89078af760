"""Oracle digests of every BASELINE config at full size (test infrastructure).

    python tools/oracle_digests.py [--configs C2,C3,...] [--cache oracle_cache]

Runs ONLY the plain CPU oracle (oracle/posit_oracle.c through oracle/oracle.py)
on the seeded BASELINE inputs (synthetic_inputs.py) and writes, per config,
``tests/golden/config_digests/<cfg>.json`` with

* ``input_sha256``    SHA-256 of the posit32 input words (oracle converter),
* ``oracle_sha256``   SHA-256 of oracle/posit_oracle.c (the oracle version),
* ``output_sha256``   SHA-256 of the whole output (matrix words, row-major,
                      then ipiv int32, then info int32 -- all little endian),
* ``row_digests``     per output row: the first 8 bytes (16 hex digits) of
                      SHA-256(row words), so a GPU mismatch is located to a row,
* ``ipiv_sha256``, ``info``, timing, host core count.

Nothing here reads the CUDA path: no value comes from the GPU.  The raw oracle
outputs are cached (gitignored) under ``--cache`` keyed by config, input
SHA-256 and oracle SHA-256 ("oracle result caching").

Configs (BASELINE.json configs[0..4]; SURVEY 8(d) recipes):
  C1      LU n=256 (or_getrf)
  C2      GEMM C <- C - A B, 4096^3 (or_gemm 'N','N', alpha=-1, beta=+1)
  C3      Cholesky lower n=8192 (or_potrf_lower); the upper triangle is the
          input's, unchanged
  C4      LU n=16384 (or_getrf)
  C5m16, C5m4, C5p0, C5p4, C5p16   LU n=8192 on U[-1,1) * 2^s
The blocked GPU factorisations (any nb, any rank count) must reproduce the
unblocked oracle bit for bit by the order contract (reading Q6).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic_inputs as SI  # noqa: E402
from oracle import oracle as O  # noqa: E402

OUT_DIR = os.path.join(ROOT, "tests", "golden", "config_digests")
C5_NAMES = {"C5m16": -16, "C5m4": -4, "C5p0": 0, "C5p4": 4, "C5p16": 16}
ALL = ["C1", "C2", "C3"] + list(C5_NAMES) + ["C4"]


def sha256(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def row_digests(M: np.ndarray) -> list[str]:
    M = np.ascontiguousarray(M, dtype=np.uint32)
    return [hashlib.sha256(M[i].tobytes()).hexdigest()[:16] for i in range(M.shape[0])]


def oracle_sha() -> str:
    with open(os.path.join(ROOT, "oracle", "posit_oracle.c"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def inputs(cfg: str):
    """Posit32 input words of a config, converted by the ORACLE's from_f64."""
    if cfg == "C1":
        return {"A": O.from_f64_array(SI.config1())}
    if cfg == "C2":
        A, B, C = SI.config2()
        return {"A": O.from_f64_array(A), "B": O.from_f64_array(B), "C": O.from_f64_array(C)}
    if cfg == "C3":
        return {"A": O.from_f64_array(SI.config3())}
    if cfg == "C4":
        return {"A": O.from_f64_array(SI.config4())}
    return {"A": O.from_f64_array(SI.config5(C5_NAMES[cfg]))}


def run_lu_resumable(cfg: str, A0: np.ndarray, in_sha: str, ckpt_dir: str, budget_s: float, chunk: int = 64,
                     partial_path: str | None = None, ckpt_every: float = 0.0, stop_after_chunks: int = 0):
    """The textbook LU in chunks of `chunk` steps (or_getrf_steps: the same loop),
    checkpointed to ckpt_dir (A, ipiv, info, next step) when the time budget
    would run out; resumes from a checkpoint of the same input.  -> (LU, ipiv,
    info) or None if stopped at a checkpoint."""
    t0 = t_call = time.time()
    os.makedirs(ckpt_dir, exist_ok=True)
    base = os.path.join(ckpt_dir, f"{cfg}_{in_sha[:16]}")
    if os.path.exists(base + ".json"):
        st = json.load(open(base + ".json"))
        k = st["k"]
        A = np.load(base + f"_A_{k}.npy")
        ipiv = np.load(base + f"_ipiv_{k}.npy")
        info = np.array([st["info"]], np.int32)
        t0 -= st.get("elapsed", 0.0)                 # report the whole run's oracle time
        print(f"{cfg}: resuming at step {k} of {A.shape[0]} (checkpoint)", flush=True)
    else:
        A, ipiv, info, k = A0.copy(), np.zeros(min(A0.shape), np.int32), np.zeros(1, np.int32), 0
    kmax = min(A.shape)
    last = 0.0
    t_ck = time.time()
    chunks_done = 0
    while k < kmax:
        stop = (budget_s > 0 and time.time() - t_call + 1.3 * last + 30 > budget_s) or \
               (stop_after_chunks > 0 and chunks_done >= stop_after_chunks)      # the latter: tests
        if stop or (ckpt_every > 0 and time.time() - t_ck > ckpt_every and k > 0):
            # the arrays of step k under their own names, then the index (.json) renamed into
            # place: a kill at any point leaves the previous checkpoint whole
            np.save(base + f"_A_{k}.npy", A)
            np.save(base + f"_ipiv_{k}.npy", ipiv)
            json.dump({"k": k, "info": int(info[0]), "elapsed": time.time() - t0}, open(base + ".tmp.json", "w"))
            os.replace(base + ".tmp.json", base + ".json")
            for f in os.listdir(ckpt_dir):
                if f.startswith(os.path.basename(base) + "_") and f.endswith(".npy") and not f.endswith(f"_{k}.npy"):
                    os.remove(os.path.join(ckpt_dir, f))
            t_ck = time.time()
            print(f"{cfg}: checkpoint at step {k} of {kmax} after {time.time() - t0:.0f} s", flush=True)
            if partial_path:
                # Right-looking LU: after steps 0..k-1, output rows 0..k-1 (U's row and the
                # L entries left of the diagonal) and ipiv[0..k-1] are final -- later steps
                # swap and update rows >= k only.  Their digests are already the full run's.
                json.dump({"config": cfg, "partial_rows": k, "of_rows": int(A.shape[0]), "input_sha256": in_sha,
                           "oracle_sha256": oracle_sha(), "ipiv_head_sha256": sha256(ipiv[:k]),
                           "info_so_far": int(info[0]), "oracle_seconds": round(time.time() - t0, 1),
                           "oracle_threads": O.num_threads(), "host": platform.node(),
                           "digest_rule": "row i < partial_rows: sha256(row-major uint32 LE words of row i)[:16 hex]",
                           "row_digests": row_digests(A[:k])}, open(partial_path + ".tmp", "w"), indent=0)
                os.replace(partial_path + ".tmp", partial_path)
            if stop:
                return None
        tc = time.time()
        O.getrf_steps(A, ipiv, info, k, min(kmax, k + chunk))
        last = time.time() - tc
        k = min(kmax, k + chunk)
        chunks_done += 1
    for f in os.listdir(ckpt_dir):
        if f.startswith(os.path.basename(base)):
            os.remove(os.path.join(ckpt_dir, f))
    return A, ipiv, int(info[0]), time.time() - t0


def run(cfg: str, X: dict):
    """-> (output matrix, ipiv or None, info or None, op description)."""
    if cfg == "C2":
        return O.gemm(X["A"], X["B"], X["C"]), None, None, "or_gemm('N','N', alpha=-1, beta=+1)"
    if cfg == "C3":
        L, info = O.potrf_lower(X["A"])
        return L, None, info, "or_potrf_lower (unblocked; upper triangle untouched)"
    LU, ipiv, info = O.getrf(X["A"])
    return LU, ipiv, info, "or_getrf (unblocked right-looking kij, partial pivoting)"


T_START = time.time()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(ALL))
    ap.add_argument("--out-dir", default=OUT_DIR)
    ap.add_argument("--cache", default=os.path.join(ROOT, "oracle_cache"))
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ckpt-dir", default=None, help="LU configs: checkpoint / resume directory")
    ap.add_argument("--time-budget", type=float, default=0.0, help="seconds; checkpoint and stop before it runs out")
    ap.add_argument("--ckpt-every", type=float, default=0.0, help="seconds between periodic checkpoints (0: only at the budget)")
    args = ap.parse_args()
    os.makedirs(args.out_dir, exist_ok=True)
    os.makedirs(args.cache, exist_ok=True)
    osha = oracle_sha()
    for cfg in args.configs.split(","):
        cfg = cfg.strip()
        X = inputs(cfg)
        in_sha = sha256(*[X[k] for k in sorted(X)])
        out_path = os.path.join(args.out_dir, f"{cfg}.json")
        if not args.force and os.path.exists(out_path):
            old = json.load(open(out_path))
            if old.get("input_sha256") == in_sha and old.get("oracle_sha256") == osha:
                print(f"{cfg}: up to date", flush=True)
                continue
        print(f"{cfg}: running oracle on {O.num_threads()} threads ...", flush=True)
        t0 = time.time()
        if args.ckpt_dir and cfg not in ("C2", "C3"):
            left = args.time_budget - (time.time() - T_START) if args.time_budget > 0 else 0.0
            r = run_lu_resumable(cfg, X["A"], in_sha, args.ckpt_dir, left,
                                  partial_path=os.path.join(args.out_dir, f"{cfg}_partial.json"),
                                  ckpt_every=args.ckpt_every)
            if r is None:
                sys.exit(2)
            M, ipiv, info, dt_total = r
            what = "or_getrf (unblocked right-looking kij, partial pivoting; run as or_getrf_steps chunks)"
        else:
            M, ipiv, info, what = run(cfg, X)
            dt_total = time.time() - t0
        dt = dt_total
        parts = [M] + ([ipiv] if ipiv is not None else []) + ([np.array([info], np.int32)] if info is not None else [])
        rec = {
            "config": cfg,
            "op": what,
            "shape": list(M.shape),
            "input_sha256": in_sha,
            "input_sha256_parts": {k: sha256(X[k]) for k in sorted(X)},
            "oracle_sha256": osha,
            "output_sha256": sha256(*parts),
            "matrix_sha256": sha256(M),
            "ipiv_sha256": sha256(ipiv) if ipiv is not None else None,
            "info": info,
            "oracle_seconds": round(dt, 1),
            "oracle_threads": O.num_threads(),
            "host": platform.node(),
            "digest_rule": "row i: sha256(row-major uint32 LE words of row i)[:16 hex]; "
                           "output_sha256 = sha256(matrix || ipiv int32 || info int32)",
            "row_digests": row_digests(M),
        }
        key = f"{cfg}_{in_sha[:12]}_{osha[:12]}"
        np.save(os.path.join(args.cache, key + ".npy"), M)
        if ipiv is not None:
            np.save(os.path.join(args.cache, key + "_ipiv.npy"), ipiv)
        with open(out_path, "w") as f:
            json.dump(rec, f, indent=0)
        print(f"{cfg}: done in {dt:.0f} s, output {rec['output_sha256'][:16]}", flush=True)


if __name__ == "__main__":
    main()
