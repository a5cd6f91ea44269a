"""Kernel time of one config at several CTAs/SM (plain build), for the ncu occupancy probe.

    python scripts/occ_probe.py C5 2 4 7        # prints ctas, kernel ms (best of 3)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_05039_b200 import MBEGraph  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402

with MBEGraph.from_graph(I.config_graph(sys.argv[1])) as G:
    for c in [int(x) for x in sys.argv[2:]]:
        ms = [G.enumerate(ctas_per_sm=c).kernel_ms for _ in range(int(os.environ.get("REPS", "3")))]
        print(c, round(min(ms), 2), flush=True)
