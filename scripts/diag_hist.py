"""MBE_STATS diagnostics for one config (stderr histograms; MBE_DEBUG_HIST=1 MBE_DEBUG_LONGEST=1).

    MBE_DEBUG_HIST=1 MBE_DEBUG_LONGEST=1 python scripts/diag_hist.py C5
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_05039_b200 import MBE_STATS, MBEGraph  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402

for cfg in sys.argv[1:]:
    with MBEGraph.from_graph(I.config_graph(cfg)) as G:
        plain = [G.enumerate().kernel_ms for _ in range(3)]
        print(f"== {cfg}: plain kernel ms {[round(x, 2) for x in plain]}", file=sys.stderr, flush=True)
        r = G.enumerate(flags=MBE_STATS)
        tot = r.n_warps * r.kernel_ms * 1.965e6
        print(f"== {cfg}: count {r.count} tasks {r.tasks} frames {r.frames} list {r.list_tasks} stats kernel "
              f"{r.kernel_ms:.2f} ms alg {r.alg_parts} phase% {[round(100 * c / tot, 1) for c in r.phase_cycles]}",
              file=sys.stderr, flush=True)
