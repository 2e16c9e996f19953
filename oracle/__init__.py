"""CPU oracle for the OWQ hot path -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  See owq_oracle.py.
"""
from .owq_oracle import *  # noqa: F401,F403
from .owq_oracle import __all__  # noqa: F401
