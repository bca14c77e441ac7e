"""CPU oracle for the Clifford conv / multivector-activation hot path.

TEST INFRASTRUCTURE ONLY. Nothing in the product package
(`paper_2507_01040_b200/`) may import, call or link this package; only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` use it, and only as the checker or as the timed
CPU baseline.

Parity pin: the restatement is checked against golden vectors produced by
importing the reference package (`mvkernels`, /root/reference/pkg/src) in the
build container; see `tests/golden/make_golden.py` and
`tests/test_oracle_golden.py`.
"""

from .oracle import *  # noqa: F401,F403
