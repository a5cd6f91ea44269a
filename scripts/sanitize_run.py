"""Workload for compute-sanitizer (memcheck / synccheck) and for the race-stress build.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py [--graphs 50] [--reps 1]
    MBE_LIB_PATH=variants/delays.so python scripts/sanitize_run.py --graphs 200 --reps 5

C1 (crown 12, G(200,200,0.05)) and seeded random graphs, each under the default (single-task
steals), steal-half, the deferred Step 3 (defer_min = 1) and a shared claim counter, every result
compared with the CPU oracle (count, hash, tasks, pruned).  Exits nonzero on the first mismatch.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import reference as R  # noqa: E402
from paper_2401_05039_b200 import MBE_STEAL_HALF, ClaimCounter, MBEGraph  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402


def graphs(n):
    yield I.crown(12)
    yield I.erdos_renyi_c1b()
    ps = [0.05, 0.1, 0.3, 0.5]
    for k in range(n):
        z = R.mix64(0x5A17 + k)
        n1, n2 = 20 + z % 300, 20 + (z >> 12) % 300
        yield I.random_bipartite(n1, n2, ps[k % 4] if n1 * n2 < 20000 else 0.04, 777 + k)
    # wide (8/16-word) bit rows and hub list frames
    yield I.random_bipartite(30, 500, 0.5, 6)
    yield I.random_bipartite(12, 400, 0.7, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graphs", type=int, default=50)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    ctr = ClaimCounter(0)
    runs = 0
    for g in graphs(a.graphs):
        want = oracle.mbea(g)
        key = (want.count, want.hash, want.tasks, want.pruned)
        with MBEGraph.from_graph(g) as G:
            for _ in range(a.reps):
                for cfg in (dict(), dict(flags=MBE_STEAL_HALF), dict(defer_min=1), dict(ctas_per_sm=1, threads_per_cta=64)):
                    r = G.enumerate(**cfg)
                    got = (r.count, r.hash, r.tasks, r.pruned)
                    runs += 1
                    if got != key:
                        print(f"MISMATCH {g.name} {cfg}: {got} != {key}", flush=True)
                        sys.exit(1)
                ctr.reset()
                r0 = G.enumerate(rank=0, world=2, claim_counter=ctr.ptr, arena_bytes=4096, flags=0x40)
                r1 = G.enumerate(rank=1, world=2, claim_counter=ctr.ptr, arena_bytes=4096, flags=0x40)
                runs += 2
                if (r0.count + r1.count, (r0.hash + r1.hash) & R.MASK64) != (want.count, want.hash):
                    print(f"MISMATCH shared counter {g.name}", flush=True)
                    sys.exit(1)
    ctr.close()
    print(f"OK {runs} enumerations, all equal to the oracle", flush=True)


if __name__ == "__main__":
    main()
