"""CPU oracle for the halfgnn hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package halfsparse (arXiv 2411.01109's
artifact, /root/reference/pkg/src/halfsparse) for the operators on the hot
path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import it, and only as the checker or the timed CPU
baseline.  The product package (paper_2411_01109_b200) never imports it.

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the real reference (tests/golden/make_golden.py,
run in the build container where the reference is importable).
"""
from .halfgnn_oracle import *  # noqa: F401,F403
