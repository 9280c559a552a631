"""fp64 CPU oracle of MoA attention -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  See moa_oracle.py.
"""
from .moa_oracle import *  # noqa: F401,F403
from .moa_oracle import __all__  # noqa: F401
