"""The chunked / checkpointed oracle LU of tools/oracle_digests.py (CPU only).

C4's oracle run is longer than one GPU-box call, so it runs as or_getrf_steps
chunks with checkpoints, and a stopped run publishes the digests of the rows
that are already final.  Checked here on a small matrix: (1) the resumed run
equals the one-shot or_getrf bit for bit; (2) after k steps rows < k and
ipiv[:k] are final, i.e. their digests equal the finished run's.
"""
import hashlib
import json
import os
import sys

import numpy as np

import synthetic_inputs as SI
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle_digests as D  # noqa: E402


def test_chunked_lu_equals_one_shot_and_partial_rows_are_final(tmp_path):
    n = 96
    A = O.from_f64_array(SI.lu_matrix(n, 5))
    ref, rpiv, rinfo = O.getrf(A)
    in_sha = D.sha256(A)
    ck, part = str(tmp_path / "ck"), str(tmp_path / "P_partial.json")
    r = D.run_lu_resumable("P", A, in_sha, ck, 0.0, chunk=40, partial_path=part, stop_after_chunks=1)
    assert r is None
    p = json.load(open(part))
    k = p["partial_rows"]
    assert k == 40 and p["of_rows"] == n and p["input_sha256"] == in_sha
    rows = [hashlib.sha256(ref[i].tobytes()).hexdigest()[:16] for i in range(n)]
    assert p["row_digests"] == rows[:k]                      # rows < k are already the final rows
    assert p["ipiv_head_sha256"] == D.sha256(rpiv[:k])
    st = json.load(open(os.path.join(ck, f"P_{in_sha[:16]}.json")))
    mid = np.load(os.path.join(ck, f"P_{in_sha[:16]}_A_{st['k']}.npy"))
    assert np.array_equal(mid[:k], ref[:k]) and not np.array_equal(mid[k:], ref[k:])
    # resume with periodic checkpoints on: same bits as the one-shot run, checkpoint files removed
    M, ipiv, info, _ = D.run_lu_resumable("P", A, in_sha, ck, 0.0, chunk=16, partial_path=part, ckpt_every=1e-9)
    assert np.array_equal(M, ref) and np.array_equal(ipiv, rpiv) and info == rinfo
    assert os.listdir(ck) == []


DIG = os.path.join(ROOT, "tests", "golden", "config_digests")
SHAPES = {"C1": 256, "C2": 4096, "C3": 8192, "C4": 16384, "C5m16": 8192, "C5m4": 8192, "C5p0": 8192, "C5p4": 8192,
          "C5p16": 8192}


def _versions():
    return {l.split()[0] for l in open(os.path.join(DIG, "ORACLE_VERSIONS.txt")) if l[:1] not in "# \n"}


def test_committed_digests_are_well_formed_and_name_a_listed_oracle_version():
    names = sorted(f[:-5] for f in os.listdir(DIG) if f.endswith(".json"))
    assert {"C1", "C2", "C3", "C5m16", "C5m4", "C5p0", "C5p4", "C5p16"} <= set(names)
    for name in names:
        d = json.load(open(os.path.join(DIG, name + ".json")))
        cfg = d["config"]
        assert d["oracle_sha256"] in _versions(), name
        n = SHAPES[cfg]
        rows = d["partial_rows"] if name.endswith("_partial") else n
        assert len(d["row_digests"]) == rows and all(len(x) == 16 for x in d["row_digests"]), name
        assert len(d["input_sha256"]) == 64
        if not name.endswith("_partial"):
            assert d["shape"] == [n, n] and len(d["output_sha256"]) == 64


def test_c1_digest_reproduces_from_the_oracle():
    """The committed C1 digest is what tools/oracle_digests.py computes today from oracle/ alone
    (input by the oracle's converter, output by or_getrf): the digest rule end to end."""
    d = json.load(open(os.path.join(DIG, "C1.json")))
    X = D.inputs("C1")
    assert D.sha256(X["A"]) == d["input_sha256"]
    LU, ipiv, info = O.getrf(X["A"])
    assert D.row_digests(LU) == d["row_digests"] and D.sha256(ipiv) == d["ipiv_sha256"] and info == d["info"]
    assert D.sha256(LU, ipiv, np.array([info], np.int32)) == d["output_sha256"]


def test_c5_inputs_are_exact_power_of_two_scalings_of_one_draw():
    """configs[4]: the five shifts share one U[-1,1) draw (np.ldexp is exact), and the committed
    digests were taken on exactly these inputs (input SHA-256 by the oracle's converter)."""
    for name, s in D.C5_NAMES.items():
        d = json.load(open(os.path.join(DIG, name + ".json")))
        assert D.sha256(O.from_f64_array(SI.config5(s))) == d["input_sha256"], name
