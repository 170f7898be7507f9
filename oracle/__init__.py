"""CPU oracle (TEST INFRASTRUCTURE ONLY) — see phe_oracle.py's header.

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  The product package never imports it.
"""
from . import phe_oracle  # noqa: F401
from .phe_oracle import PAPER, TOY, Params  # noqa: F401
