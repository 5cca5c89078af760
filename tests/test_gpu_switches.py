"""Every traversal switch and every GEMM tile instantiation against the oracle.

The library reads its POSIT_* switches once per process (DESIGN.md section 8,
"Run-time switches"), so each setting runs tests/switch_worker.py in a fresh
subprocess on the same inputs; the parent compares its outputs word by word
with the CPU oracle.  By the order contract (reading Q6) every switch changes
only the traversal, so all of them must give the oracle's bits:

* GEMM: POSIT_GEMM_VARIANT 11..14 (the integer-MAC tiles G1..G4), 21..24 (the
  binary64-pipe tiles D1..D4) and POSIT_GEMM_PATH=0 (integer MAC by default) x
  {NN, NT, TN, SYRK} at a shape above the one-thread-per-output cutoff with
  ragged tails in m, n and k, plus the default model choice and the tiny-kernel
  routes (POSIT_GEMM_TINY = 0 / 2);
* LU and Cholesky (n = 1100, nb = 256: blocked steps with lookahead, then the
  fused tail): lookahead off, programmatic dependent launch off, the leaf
  variants, the U12 in-block kernels, the Cholesky TRSM variants, the
  recursive potf2, no fused tail, and forced GEMM tiles.  The serial /
  non-PDL / non-lookahead runs double as the race check the missing
  compute-sanitizer would give: the concurrent schedule must equal them.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import synthetic_inputs as SI
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "switch_worker.py")
M, N, K = 300, 520, 70          # above the tiny cutoff (m n > 65536), ragged vs 64 x 128 x 16 tiles
NS = 330                         # SYRK order
NL = 1100                        # LU / Cholesky order: 3 blocked steps + fused tail (LU), 5 steps (Cholesky)


def _run_worker(tmp_path, job, inputs, env_extra, tag):
    src = tmp_path / f"in_{job}.npz"
    if not src.exists():
        np.savez(src, **inputs)
    dst = tmp_path / f"out_{job}_{tag}.npz"
    env = dict(os.environ)
    for k in [k for k in env if k.startswith("POSIT_") and k != "POSIT_LIB_PATH"]:
        del env[k]
    env.update(env_extra)
    r = subprocess.run([sys.executable, WORKER, str(src), str(dst), job], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(dst)


@pytest.fixture(scope="module")
def gemm_case():
    A64, B64, C64 = SI.config2(n=N, m=M, k=K)
    A, B, C = O.from_f64_array(A64), O.from_f64_array(B64), O.from_f64_array(C64)
    As = O.from_f64_array(SI.normal_matrix((NS, K), 1.0, 22))
    S = O.from_f64_array(SI.normal_matrix((NS, NS), 1.0, 21))
    inputs = {"A": A, "B": B, "Bt": B.T.copy(), "At": A.T.copy(), "C": C, "As": As, "S": S}
    ref = {"nn": O.gemm(A, B, C), "nt": O.gemm(A, B.T.copy(), C, transb="T"),
           "tn": O.gemm(A.T.copy(), B, C, transa="T"), "syrk": O.syrk_lower(As, S)}
    return inputs, ref


GEMM_VARIANTS = [{}, {"POSIT_GEMM_VARIANT": "11"}, {"POSIT_GEMM_VARIANT": "12"}, {"POSIT_GEMM_VARIANT": "13"},
                 {"POSIT_GEMM_VARIANT": "14"}, {"POSIT_GEMM_TINY": "0"}, {"POSIT_GEMM_PATH": "0"},
                 {"POSIT_GEMM_VARIANT": "21"}, {"POSIT_GEMM_VARIANT": "22"}, {"POSIT_GEMM_VARIANT": "23"},
                 {"POSIT_GEMM_VARIANT": "24"}, {"POSIT_GEMM_VARIANT": "22", "POSIT_GEMM_TINY": "0"}]


@pytest.mark.parametrize("env", GEMM_VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_gemm_syrk_variants_match_oracle(cuda_ok, tmp_path, gemm_case, env):
    inputs, ref = gemm_case
    tag = "_".join(f"{k}{v}" for k, v in env.items()) or "default"
    out = _run_worker(tmp_path, "gemm", inputs, env, tag)
    for name in ("nn", "nt", "tn"):
        assert int(np.count_nonzero(out[name] != ref[name])) == 0, (name, env)
    il, iu = np.tril_indices(NS), np.triu_indices(NS, 1)
    assert int(np.count_nonzero(out["syrk"][il] != ref["syrk"][il])) == 0, ("syrk", env)
    assert int(np.count_nonzero(out["syrk"][iu] != inputs["S"][iu])) == 0, "SYRK touched the upper triangle"


@pytest.fixture(scope="module")
def lapack_case():
    L = O.from_f64_array(SI.config4(NL))        # configs[3] recipe at n = 1100
    P = O.from_f64_array(SI.config3(NL))        # configs[2] recipe at n = 1100
    lu, ipiv, info = O.getrf(L)
    chol, cinfo = O.potrf_lower(P)
    assert info == 0 and cinfo == 0
    return {"L": L, "P": P}, lu, ipiv, chol


LAPACK_SWITCHES = [
    {},
    {"POSIT_LOOKAHEAD": "0"},
    {"POSIT_PDL": "0"},
    {"POSIT_LOOKAHEAD": "0", "POSIT_PDL": "0", "POSIT_TAIL_W": "0"},
    {"POSIT_LEAF_COOP": "0"},
    {"POSIT_LEAF_COOP": "2"},
    {"POSIT_PANEL_LEAF": "64"},
    {"POSIT_LEAF_CTAS": "16"},
    {"POSIT_LEAF_DDIV": "1"},
    # one 1024-thread CTA per side-stream leaf, never the wide leaf on the side stream: tall CTAs
    # (>= 512 rows in the first lookahead panels), where the row-mode update applies
    {"POSIT_WIDE_LEAF_COLS": "0", "POSIT_SIDE_LEAF_CTAS": "1"},
    {"POSIT_LEAF_ROWS": "1", "POSIT_WIDE_LEAF_COLS": "0", "POSIT_SIDE_LEAF_CTAS": "1"},
    {"POSIT_LEAF_ROWS": "1", "POSIT_LEAF_DDIV": "1", "POSIT_WIDE_LEAF_COLS": "0", "POSIT_SIDE_LEAF_CTAS": "1"},
    {"POSIT_LEAF_ROWS": "1", "POSIT_LEAF_DDIV": "1"},
    {"POSIT_LEAF_DDIV": "1", "POSIT_LEAF_CTAS": "16"},
    {"POSIT_LLNU_D": "0", "POSIT_LLNU_G8": "0", "POSIT_LLNU_COL": "0", "POSIT_LLNU_BLK": "32"},
    {"POSIT_LLNU_D": "0", "POSIT_LLNU_G8": "0", "POSIT_LLNU_COL": "8"},
    {"POSIT_LLNU_D": "0", "POSIT_LLNU_G8": "0"},
    {"POSIT_LLNU_D": "0"},
    {"POSIT_RLTN": "8,16"},
    {"POSIT_RLTN": "16,32"},
    {"POSIT_RLTN": "16,16,128"},
    {"POSIT_RLTN_D": "0"},
    {"POSIT_POTF2": "0"},
    {"POSIT_POTF2": "1"},
    {"POSIT_POTF2_NC": "8"},
    {"POSIT_POTF2_DEFER": "1"},
    {"POSIT_POTF2_DEFER": "1", "POSIT_POTF2_NC": "8"},
    {"POSIT_POTF2_DDIV": "0"},
    {"POSIT_POTF2_DDIV": "1"},
    {"POSIT_POTF2_DDIV": "1", "POSIT_POTF2_NC": "8"},
    {"POSIT_POTF2_DDIV": "1", "POSIT_POTF2_DEFER": "1"},
    {"POSIT_GEMM_VARIANT": "12", "POSIT_GEMM_TINY": "2"},
    {"POSIT_GEMM_VARIANT": "13"},
    {"POSIT_GEMM_VARIANT": "14"},
    {"POSIT_GEMM_PATH": "0"},
    {"POSIT_GEMM_PATH": "0", "POSIT_LOOKAHEAD": "0"},
]


@pytest.mark.parametrize("env", LAPACK_SWITCHES, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_lapack_switches_match_oracle(cuda_ok, tmp_path, lapack_case, env):
    inputs, lu, ipiv, chol = lapack_case
    tag = "_".join(f"{k}{v}".replace(",", "-") for k, v in env.items()) or "default"
    out = _run_worker(tmp_path, "lapack", inputs, env, tag)
    assert int(out["lu_info"][0]) == 0 and int(out["chol_info"][0]) == 0
    assert np.array_equal(out["ipiv"], ipiv), env
    assert int(np.count_nonzero(out["lu"] != lu)) == 0, env
    il = np.tril_indices(NL)
    assert int(np.count_nonzero(out["chol"][il] != chol[il])) == 0, env
    iu = np.triu_indices(NL, 1)
    assert int(np.count_nonzero(out["chol"][iu] != inputs["P"][iu])) == 0, "upper triangle touched"
