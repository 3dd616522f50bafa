"""CPU oracle for the Mamba-2 SSD hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference engine's arithmetic
(``/root/reference/pkg/src/ssd_engine``) so that the CUDA product path can be
checked against it.  It is imported only by ``tests/``, by
``__graft_entry__.smoke()`` (as the checker) and by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs (as the timed CPU path).  The
product package ``paper_2603_09555_b200`` never imports it and has no CPU
fallback.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the *real* reference (``tests/golden/make_golden.py``
imports ``ssd_engine`` from ``/root/reference/pkg/src`` and writes the
fixtures), so parity is pinned to the reference itself, not to this
restatement.
"""

from .mamba2_cpu import *  # noqa: F401,F403
from .mamba2_cpu import __all__  # noqa: F401
