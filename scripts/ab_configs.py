"""A/B kernel timing of build variants: for each config, 1 warm-up + N plain enumerations (CUDA-event
kernel ms), checked bit-exact against the oracle golden (tests/golden/configs.txt).

    MBE_LIB_PATH=variants/x.so python scripts/ab_configs.py C2 C5 [--reps 3] [--tag x]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_05039_b200 import MBEGraph  # noqa: E402
from paper_2401_05039_b200 import inputs as I  # noqa: E402


def golden():
    rows = {}
    for line in open(os.path.join(ROOT, "tests", "golden", "configs.txt")):
        if line.strip() and not line.startswith("#"):
            f = line.split()
            rows[f[0]] = (int(f[1]), int(f[2], 16), int(f[3]), int(f[4]))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default=os.environ.get("MBE_LIB_PATH", "default"))
    ap.add_argument("--T", type=int, default=0)
    a = ap.parse_args()
    gold = golden()
    for c in a.configs:
        with MBEGraph.from_graph(I.config_graph(c)) as G:
            G.enumerate(bitmap_threshold=a.T)
            ms, ok = [], True
            for _ in range(a.reps):
                r = G.enumerate(bitmap_threshold=a.T)
                ms.append(round(r.kernel_ms, 3))
                if c in gold and (r.count, r.hash, r.tasks, r.pruned) != gold[c]:
                    ok = False
            print(json.dumps({"tag": a.tag, "config": c, "kernel_ms": ms, "min": min(ms), "exact": ok,
                              "n_warps": r.n_warps}), flush=True)


if __name__ == "__main__":
    main()
