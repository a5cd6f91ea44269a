"""Two plain enumerations of a config (no MBE_STATS) for ncu: capture the second launch.

    ncu ... -k regex:mbe_search_kernel -s 1 -c 1 python scripts/profile_run.py C2
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_05039_b200 import MBEGraph  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402

with MBEGraph.from_graph(I.config_graph(sys.argv[1] if len(sys.argv) > 1 else "C2")) as G:
    for _ in range(2):
        r = G.enumerate()
    print(r.count, hex(r.hash), r.kernel_ms)
