"""CPU oracle for the RPLU pivot loop — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithms (arXiv 2601.22344, package
``rplu`` 0.1.0 under /root/reference/pkg/src/rplu), each function citing the
file:line it follows.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it,
and only as the checker or the timed CPU baseline — never as the product path.
The product (``paper_2601_22344_b200``) has no CPU fallback.

Parity pin: the restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.
"""

from .rplu_oracle import *  # noqa: F401,F403
from . import consumers_oracle as consumers  # noqa: F401,E402  (§8(f4) consumers)
from . import plan_oracle as plan  # noqa: F401,E402  (§8(f1) certified bounds)
