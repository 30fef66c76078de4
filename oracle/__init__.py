"""CPU oracle for the FastGL per-mini-batch hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference package
``minigl`` 0.1.0 (``/root/reference/pkg/src/minigl``) for every row of
SURVEY.md section 8(a).  Each function cites the reference file:line it follows.

Rules (DESIGN.md section "Oracle"):

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import this package, and
  only as the checker or the timed CPU baseline -- never as the product path.
  The product package ``paper_2409_14939_b200`` never imports it.
* Parity is pinned: ``tests/test_oracle_golden.py`` checks every function
  here against golden vectors produced by running the unmodified reference
  (``tests/golden/make_golden.py``, committed with its outputs).
* Third-party arithmetic on the path is numpy's Philox4x64-10 stream
  (numpy 2.3.5, pinned ``numpy>=1.24`` in ``pkg/pyproject.toml:10-13``).  It is
  restated bit-exactly in :mod:`oracle.philox` and checked against numpy's
  own ``Generator(Philox(seed)).random``.
"""

from . import philox  # noqa: F401
from .minigl_oracle import *  # noqa: F401,F403
