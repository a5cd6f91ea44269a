"""Multi-process host logic of the multi-GPU path on CPU (gloo, world size 2):
the final (count, hash) all-reduce through 16-bit limbs, max-over-ranks timing,
and that rank shares of the level-1 subtrees (oracle per-root results) sum to
the whole."""
import os
import random
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import bench

MASK64 = (1 << 64) - 1


def test_limbs_roundtrip_and_sum():
    rng = random.Random(3)
    for _ in range(200):
        vals = [(rng.getrandbits(64), rng.getrandbits(64)) for _ in range(8)]
        assert bench.from_limbs(bench.limbs_of(*vals[0])) == vals[0]
        summed = [sum(col) for col in zip(*[bench.limbs_of(c, h) for c, h in vals])]
        want = (sum(c for c, _ in vals) & MASK64, sum(h for _, h in vals) & MASK64)
        assert bench.from_limbs(summed) == want


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shares, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, h = shares[rank]
    out[rank] = (bench.allreduce_result(c, h, "cpu"), bench.max_over_ranks(float(rank + 1) * 1.5, "cpu"))
    dist.destroy_process_group()


def test_gloo_world2_allreduce_and_max():
    import oracle
    from paper_2401_05039_b200 import inputs as I

    g = I.erdos_renyi_c1b()
    tot = oracle.mbea(g)
    pr = oracle.mbea_roots(g, np.arange(g.n2), candidate_side=2)
    # rank r takes every world-th subtree (any partition of the level-1 subtrees sums to the whole)
    world = 2
    shares = []
    for r in range(world):
        part = pr[r::world]
        shares.append((int(part[:, 0].sum()), int(part[:, 1].astype(object).sum()) & MASK64))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, shares, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(world):
        (c, h), mx = out[r]
        assert (c, h) == (tot.count, tot.hash)
        assert mx == 3.0
