"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY — see oracle/dit.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg.  Never imported by the product package.
"""
from . import dit  # noqa: F401
