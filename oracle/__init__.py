"""CPU oracle for the MO-FEM solve path — TEST INFRASTRUCTURE ONLY.

This package is a plain numpy/scipy restatement of the reference algorithm
(`sylfem`, /root/reference/pkg/src/sylfem) for the hot path named in
BASELINE.json: 1D assembly, Sylvester term lists, the LU-factorized single-term
preconditioner, the spectral (reduced) two-term solve, MO-PCG and the two IMEX
drivers.  Every function cites the reference file:line it restates.

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` — as the checker
or the timed CPU baseline, never as a product code path.  The product package
``paper_2109_01173_b200`` never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by running the reference itself in the build
container (``tests/golden/make_golden.py``), so the parity claims made
through this oracle are pinned to the reference's own outputs.
"""

from .mofem import *  # noqa: F401,F403
