"""CPU oracle for the FEAST contour-projection hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product (``paper_1203_4031_b200``) may import this package.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs use it, and only as the checker or the timed CPU
reference arm, never as the thing measured or shipped.

The oracle restates the reference algorithm (``feastlib`` 0.1.0 under
``/root/reference/pkg/src/feastlib``) in plain numpy, each function citing the
reference file:line it follows.  It is pinned against golden vectors produced
by running the reference itself in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.
"""

from .feast_oracle import *  # noqa: F401,F403
