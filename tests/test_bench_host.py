"""Host-side pieces of bench.py that need no GPU: the CPU-oracle sampling behind cpu_baseline and the
--impl reference arm (one uniform sample of level-1 subtrees, optionally split into disjoint parts)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_oracle_rate_split_sample_is_a_partition():
    import bench
    import oracle
    from paper_2401_05039_b200 import inputs as I

    oracle.build_oracle()
    g = I.erdos_renyi_c1b()
    parts = []
    rate, info = bench.oracle_rate(g, 0.2, seed=3, parts=3, part_stats=parts)
    assert len(parts) == 3 and rate > 0
    # the parts hold the whole sample: their counts sum to the sample's count
    assert sum(p[0] for p in parts) == info["count"]
    assert info["roots"] >= 3
    # the same seed draws the same sample whether or not it is split
    rate1, info1 = bench.oracle_rate(g, 0.2, seed=3)
    assert info1["count"] == info["count"] and info1["roots"] == info["roots"]


def test_oracle_rate_full_sample_count_matches_oracle():
    import bench
    import oracle
    from paper_2401_05039_b200 import inputs as I

    oracle.build_oracle()
    g = I.crown(6)
    # target large enough that k = 1: the sample is every level-1 subtree, so the count is the whole result
    _, info = bench.oracle_rate(g, 1e9, seed=1)
    assert info["k"] == 1
    assert info["count"] == oracle.mbea(g).count == 2 ** 6 - 2
