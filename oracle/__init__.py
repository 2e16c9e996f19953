"""CPU oracle for the OWQ hot path -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  See owq_oracle.py (the
default latency-favored representation) and owq_variants.py (act-order and
storage-favored variants).
"""
from .owq_oracle import *  # noqa: F401,F403
from .owq_oracle import __all__ as _a
from .owq_variants import *  # noqa: F401,F403
from .owq_variants import __all__ as _b

__all__ = list(_a) + list(_b)
