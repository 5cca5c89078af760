"""Every output word of every BASELINE config at full size against the oracle.

tests/golden/config_digests/<cfg>.json hold the CPU oracle's per-row SHA-256
digests and whole-output SHA-256 of C1..C5 (written by tools/oracle_digests.py
from oracle/ alone, keyed by input SHA-256 and oracle-source SHA-256).  This
test runs each config through the C ABI on the GPU at the size and block size
bench.py times (tests/config_parity.py), hashes every output row and compares:
mismatching rows must be 0 and the whole-output SHA-256 equal (SURVEY 8(d)
"Parity check"; north_star "bit-exact ... on every output word ... on all
five configs").  The GPU converts the inputs with its own posit_from_f64; the
input SHA-256 must equal the oracle converter's.

The schedule switches that remove concurrency (lookahead, programmatic
dependent launch) rerun the C5 s = 0, C3 and C4 factorisations in
subprocesses: the concurrent default must equal the serial schedule and the
oracle (the race check that stands in for compute-sanitizer).
"""
import json
import os
import subprocess
import sys

import pytest

from tests.config_parity import ALL, DIGESTS, compare, compare_partial

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRESENT = [c for c in ALL if os.path.exists(os.path.join(DIGESTS, f"{c}.json"))]


@pytest.mark.parametrize("cfg", PRESENT)
def test_config_every_word_matches_oracle(cuda_ok, cfg):
    rep = compare(cfg)
    assert rep["input_sha_match"], rep
    assert rep["mismatched_rows"] == 0, rep
    assert rep["ok"], rep


PARTIAL = [c for c in ALL if c not in PRESENT and os.path.exists(os.path.join(DIGESTS, f"{c}_partial.json"))]


@pytest.mark.parametrize("cfg", PARTIAL)
def test_config_final_rows_match_oracle(cuda_ok, cfg):
    """An LU config whose oracle run was checkpointed after k steps (<cfg>_partial.json):
    output rows < k (every column) and ipiv[:k] are final there and must match."""
    rep = compare_partial(cfg)
    assert rep["input_sha_match"], rep
    assert rep["mismatched_rows"] == 0 and rep["ipiv_match"], rep


SERIAL = [{"POSIT_LOOKAHEAD": "0"}, {"POSIT_PDL": "0"}, {"POSIT_LOOKAHEAD": "0", "POSIT_PDL": "0"}]


@pytest.mark.parametrize("env", SERIAL, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_config_serial_schedules_match_oracle(cuda_ok, env):
    cfgs = [c for c in ("C5p0", "C3", "C4") if c in PRESENT]
    if not cfgs:
        pytest.skip("no oracle digests for C5p0 / C3 / C4")
    full = dict(os.environ)
    full.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "config_parity.py"), "--configs", ",".join(cfgs)],
                       env=full, capture_output=True, text=True, timeout=1200)
    reps = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(reps) == len(cfgs), r.stderr[-2000:]
    for rep in reps:
        assert rep["ok"], rep
