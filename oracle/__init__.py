"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the blockwise-inversion hot path.

This package is a NumPy restatement of the reference ``blockinv`` algorithms
(`/root/reference/pkg/src/blockinv/`), written from the reference's behaviour
and cited function-by-function (file:line).  It exists to *check* the B200
product, never to *be* it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2305_11103_b200`` never imports it and has no CPU
  fallback -- it raises when its CUDA library is missing.

Parity pin: the oracle is checked against golden vectors produced by running
the reference itself in the build container (``tests/golden/make_golden.py``)
and against the reference test-suite's own known-answer tables
(``LOOPID_TABLE_B8``, ``UPDOWN_MAP_8``, ``TABLE_ROWS``); see
``tests/test_oracle.py``.
"""

from .blockinv_oracle import *  # noqa: F401,F403

