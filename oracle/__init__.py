"""oracle/ -- TEST INFRASTRUCTURE ONLY (see oracle/reference.py and oracle/csa.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
--impl reference legs may import this package.  The product path
(paper_1912_00966_b200) never imports it.
"""
from .reference import *  # noqa: F401,F403
from .reference import CSA, INF, build_oracle  # noqa: F401
