"""CPU oracle for maximal biclique enumeration — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import, call, link or execute anything here.  The
product package (paper_2401_05039_b200) never imports this package and shares
no code with it.

Contents:
  * ``mbea`` / ``mbea_roots`` / ``mbea_list`` / ``mbea_plain`` — ctypes
    wrappers around oracle/mbea_oracle.cpp, Algorithm 1
    written out with plain set copies and forward counts.
  * ``reference`` (pure Python): the result definition M(G) of P:91-98 as a
    closure brute force, Ganter's Next-Closure, and the result hash.

Parity status of each function is listed in DESIGN.md §Oracle.
"""
from .oracle import (  # noqa: F401
    OracleResult,
    build_oracle,
    mbea,
    mbea_list,
    mbea_plain,
    mbea_roots,
    mix64,
)
from . import reference  # noqa: F401
