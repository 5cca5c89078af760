"""CPU oracle for the Posit(32,2) hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import, call, link or execute
anything under ``oracle/``.  The product package ``paper_2401_14117_b200``
never does, and shares no code with it.

* ``posit_oracle.c`` / ``oracle.py`` -- plain C oracle (scalar ops and the
  textbook unblocked LU / Cholesky / GEMM in the order contract), OpenMP over
  independent output elements.
* ``checker.py`` -- exact ``Fraction`` checker that pins the C oracle.
* ``checker_wide.c`` / ``checker_wide.py`` -- checker.py's definitions with
  exact 768-bit integer comparisons (pinned to checker.py), fast enough for
  S:443's 1e7 random pairs per operation (tests/test_oracle_wide.py).
* ``make_golden.py`` -- writes ``tests/golden/`` digests by calling only the
  oracle and the seeded input generators.

Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  The
random-matrix factor bits of configs 1-5 are pinned only through the pieces
(scalar ops, special-case factorisations, invariants): the paper prints no
factor values ("parity unpinned" for those outputs beyond the pieces).
"""
