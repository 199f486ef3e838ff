"""fp64 CPU oracle for the LAKER hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product package
(paper_2604_25138_b200) never imports it and shares no code with it.
"""
from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
