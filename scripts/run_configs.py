"""Diagnostic: run the GPU path on named configs, print one JSON line each.

    python scripts/run_configs.py C2 C5 [--reps 3] [--ctas 2 --threads 256 --T 128 --flags 0]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2401_05039_b200 import MBE_STATS, MBEGraph  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--side", type=int, default=0)
    a = ap.parse_args()
    for c in a.configs:
        t = time.time()
        g = I.config_graph(c)
        tg = time.time() - t
        t = time.time()
        G = MBEGraph.from_graph(g)
        tl = time.time() - t
        cfg = dict(ctas_per_sm=a.ctas, threads_per_cta=a.threads, bitmap_threshold=a.T, candidate_side=a.side)
        st = G.enumerate(flags=a.flags | MBE_STATS, **cfg)
        times = []
        for _ in range(a.reps):
            r = G.enumerate(flags=a.flags, **cfg)
            times.append(r.kernel_ms)
        print(json.dumps(dict(config=c, count=r.count, hash=hex(r.hash), tasks=r.tasks, pruned=r.pruned,
                              steals=r.steals, kernel_ms=times, wall_ms=r.wall_ms, gen_s=round(tg, 2),
                              load_s=round(tl, 2), n_warps=r.n_warps, list_tasks=st.list_tasks,
                              bitmap_tasks=st.bitmap_tasks, frames=st.frames, alg_bytes=st.alg_bytes,
                              max_depth=st.max_depth, stats_kernel_ms=st.kernel_ms,
                              phase_frac_of_warp_time=[round(c / (st.n_warps * st.kernel_ms * 1.965e6), 4)
                                                       for c in st.phase_cycles[:16]],
                              max_task_ms=[round(c / 1.965e6, 3) for c in st.max_task_cycles],
                              roots_out_ms=round(st.roots_out_ms, 3),
                              max_phase_ms=[round(c / 1.965e6, 3) for c in st.max_phase_cycles[:16]],
                              bicliques_per_s=r.count / (min(times) / 1e3))), flush=True)
        G.close()


if __name__ == "__main__":
    main()
