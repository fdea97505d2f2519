"""CPU oracle for the sawtooth space-angle multigrid path — TEST INFRASTRUCTURE ONLY.

This package is a float64 NumPy restatement of the reference solver's
algorithm (``convsn``, arXiv 2301.09991, mounted read-only at
``/root/reference/pkg/src/convsn``).  Every function cites the reference
file:line it restates.  It is pinned against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import it, and only as the checker or the timed
CPU baseline.  The product package ``paper_2301_09991_b200`` never imports it.
"""

from .convsn_port import *  # noqa: F401,F403
from . import dense  # noqa: F401
