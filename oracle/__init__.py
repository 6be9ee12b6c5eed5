"""fp64 CPU oracle for the LaRoSA decode hot path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  Shares no code with paper_2507_01299_b200/.
"""
from .larosa_oracle import *  # noqa: F401,F403
