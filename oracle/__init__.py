"""CPU oracle for the block J-Jacobi hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_1008_4166_b200``) imports this.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may use it, and only as the checker or as the timed
CPU baseline -- never as the thing measured or shipped.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by running the reference package itself
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src``).
"""

from .jjacobi import *  # noqa: F401,F403
from .jjacobi import __all__  # noqa: F401
