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
