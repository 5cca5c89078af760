"""Full-size, every-word parity of the GPU path against the committed oracle
digests (tests/golden/config_digests/<cfg>.json, written by
tools/oracle_digests.py from the CPU oracle alone).

    python tests/config_parity.py [--configs C1,C2,...] [--digests DIR] [--out FILE]

For each BASELINE config the binary64 input is drawn from synthetic_inputs,
converted to posit32 ON THE GPU (posit_from_f64; its SHA-256 must equal the
oracle converter's, recorded as ``input_sha256``), run through the C ABI at the
configuration bench.py times (nb = 256, default switches unless the caller's
environment sets POSIT_* switches), and every output row is hashed and compared
with the oracle's row digest.  The report gives the mismatching-row count, the
first mismatching row, and the whole-output SHA-256 of both sides.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic_inputs as SI  # noqa: E402

DIGESTS = os.path.join(ROOT, "tests", "golden", "config_digests")
C5_NAMES = {"C5m16": -16, "C5m4": -4, "C5p0": 0, "C5p4": 4, "C5p16": 16}
ALL = ["C1", "C2", "C3"] + list(C5_NAMES) + ["C4"]
SWITCHES = ("POSIT_GEMM_PATH", "POSIT_LOOKAHEAD", "POSIT_PDL", "POSIT_GEMM_VARIANT", "POSIT_RLTN", "POSIT_RLTN_D", "POSIT_POTF2", "POSIT_POTF2_NC", "POSIT_POTF2_DEFER", "POSIT_POTF2_DDIV",
            "POSIT_PANEL_LEAF", "POSIT_LEAF_DDIV", "POSIT_LEAF_ROWS", "POSIT_LEAF_COOP", "POSIT_LLNU_COL", "POSIT_LLNU_G8", "POSIT_LLNU_D", "POSIT_TAIL_W")


def _sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _rows(M: np.ndarray) -> list[str]:
    return [hashlib.sha256(M[i].tobytes()).hexdigest()[:16] for i in range(M.shape[0])]


def _dev(x64: np.ndarray) -> torch.Tensor:
    import paper_2401_14117_b200 as PB
    return PB.posit_from_f64(torch.from_numpy(np.ascontiguousarray(x64)).cuda())


def _host(t: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def gpu_run(cfg: str):
    """-> (input words list, output matrix, ipiv or None, info or None, seconds)."""
    import paper_2401_14117_b200 as PB
    if cfg == "C2":
        A, B, C = SI.config2()
        dA, dB, dC = _dev(A), _dev(B), _dev(C)
        del A, B, C
        ins = {"A": _host(dA), "B": _host(dB), "C": _host(dC)}
        torch.cuda.synchronize()
        t0 = time.time()
        PB.posit_gemm(dA, dB, dC)
        torch.cuda.synchronize()
        return ins, _host(dC), None, None, time.time() - t0
    if cfg == "C3":
        dA = _dev(SI.config3())
        ins = {"A": _host(dA)}
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        t0 = time.time()
        PB.posit_potrf(dA, info, nb=SI.C3_NB)
        torch.cuda.synchronize()
        return ins, _host(dA), None, int(info.cpu()[0]), time.time() - t0
    if cfg == "C1":
        A64, nb = SI.config1(), SI.C1_NB
    elif cfg == "C4":
        A64, nb = SI.config4(), SI.C4_NB
    else:
        A64, nb = SI.config5(C5_NAMES[cfg]), SI.C5_NB
    dA = _dev(A64)
    del A64
    n = dA.shape[0]
    ins = {"A": _host(dA)}
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    t0 = time.time()
    PB.posit_getrf(dA, ipiv, info, nb=nb)
    torch.cuda.synchronize()
    return ins, _host(dA), ipiv.cpu().numpy(), int(info.cpu()[0]), time.time() - t0


def compare(cfg: str, digests_dir: str = DIGESTS) -> dict:
    path = os.path.join(digests_dir, f"{cfg}.json")
    ref = json.load(open(path))
    ins, M, ipiv, info, secs = gpu_run(cfg)
    in_sha = _sha(*[ins[k] for k in sorted(ins)])
    rows = _rows(M)
    bad = [i for i, (g, o) in enumerate(zip(rows, ref["row_digests"])) if g != o]
    parts = [M] + ([ipiv] if ipiv is not None else []) + ([np.array([info], np.int32)] if info is not None else [])
    rep = {
        "config": cfg,
        "switches": {k: os.environ[k] for k in SWITCHES if k in os.environ},
        "words_compared": int(M.size),
        "rows": len(rows),
        "input_sha_match": in_sha == ref["input_sha256"],
        "mismatched_rows": len(bad) + abs(len(rows) - len(ref["row_digests"])),
        "first_bad_row": bad[0] if bad else None,
        "ipiv_match": (ipiv is None and ref["ipiv_sha256"] is None) or
                      (ipiv is not None and _sha(ipiv) == ref["ipiv_sha256"]),
        "info": [info, ref["info"]],
        "gpu_output_sha256": _sha(*parts),
        "oracle_output_sha256": ref["output_sha256"],
        "oracle_sha256": ref["oracle_sha256"][:16],
        "gpu_seconds": round(secs, 3),
    }
    rep["ok"] = (rep["input_sha_match"] and rep["mismatched_rows"] == 0 and rep["ipiv_match"]
                 and info == ref["info"] and rep["gpu_output_sha256"] == ref["output_sha256"])
    return rep


def compare_partial(cfg: str, digests_dir: str = DIGESTS) -> dict:
    """An LU config whose oracle run stopped at a checkpoint after k steps
    (<cfg>_partial.json): output rows 0..k-1 and ipiv[0..k-1] are final there
    (later steps touch rows >= k only), so those are compared word for word."""
    ref = json.load(open(os.path.join(digests_dir, f"{cfg}_partial.json")))
    ins, M, ipiv, info, secs = gpu_run(cfg)
    k = ref["partial_rows"]
    rows = _rows(M[:k])
    bad = [i for i, (g, o) in enumerate(zip(rows, ref["row_digests"])) if g != o]
    rep = {
        "config": cfg, "partial": True, "rows_compared": k, "rows": int(M.shape[0]),
        "switches": {s: os.environ[s] for s in SWITCHES if s in os.environ},
        "words_compared": int(k * M.shape[1]),
        "input_sha_match": _sha(*[ins[s] for s in sorted(ins)]) == ref["input_sha256"],
        "mismatched_rows": len(bad) + abs(len(rows) - len(ref["row_digests"])),
        "first_bad_row": bad[0] if bad else None,
        "ipiv_match": _sha(ipiv[:k]) == ref["ipiv_head_sha256"],
        "gpu_output_sha256": _sha(M, ipiv, np.array([info], np.int32)),
        "oracle_sha256": ref["oracle_sha256"][:16], "gpu_seconds": round(secs, 3),
    }
    rep["ok"] = rep["input_sha_match"] and rep["mismatched_rows"] == 0 and rep["ipiv_match"]
    return rep


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(ALL))
    ap.add_argument("--digests", default=DIGESTS)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    reps = []
    for cfg in args.configs.split(","):
        cfg = cfg.strip()
        if not os.path.exists(os.path.join(args.digests, f"{cfg}.json")):
            if os.path.exists(os.path.join(args.digests, f"{cfg}_partial.json")):
                reps.append(compare_partial(cfg, args.digests))
            else:
                reps.append({"config": cfg, "skipped": "no oracle digest"})
        else:
            reps.append(compare(cfg, args.digests))
        print(json.dumps(reps[-1]), flush=True)
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "a") as f:
            for r in reps:
                f.write(json.dumps(r) + "\n")
    sys.exit(0 if all(r.get("ok", True) for r in reps) else 1)


if __name__ == "__main__":
    main()
