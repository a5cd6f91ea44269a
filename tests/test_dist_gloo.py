"""Multi-process host logic of the multi-GPU path on CPU (gloo, world size 2).

The rank loop of paper_2401_05039_b200/dist.py runs for real: rank 0 owns the shared counter and
zeroes it, a barrier starts every rank, each rank claims level-1 subtrees in guided-self-scheduling
chunks from the ONE shared counter (the kernel's protocol, emulated on the host over oracle per-root
results), and the (count, hash) all-reduce through 16-bit limbs gives the whole.  Also: the limb
round trip, max-over-ranks timing, and the GSS chunk schedule.
"""
import os
import random
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2401_05039_b200 import dist as D

MASK64 = (1 << 64) - 1


def test_limbs_roundtrip_and_sum():
    rng = random.Random(3)
    for _ in range(200):
        vals = [(rng.getrandbits(64), rng.getrandbits(64)) for _ in range(8)]
        assert D.from_limbs(D.limbs_of(*vals[0])) == vals[0]
        summed = [sum(col) for col in zip(*[D.limbs_of(c, h) for c, h in vals])]
        want = (sum(c for c, _ in vals) & MASK64, sum(h for _, h in vals) & MASK64)
        assert D.from_limbs(summed) == want


def test_gss_schedule_covers_every_root_once_and_shrinks():
    for n, world in [(1, 1), (7, 2), (96678, 8), (30087, 1), (5, 8)]:
        sch = D.gss_schedule(n, world)
        pos = 0
        for start, c in sch:
            assert start == pos and c >= 1
            pos += c
        assert pos == n
        sizes = [c for _, c in sch]
        assert sizes == sorted(sizes, reverse=True)  # chunks shrink as the list drains
        assert sizes[0] == D.gss_chunk(n, world) and sizes[-1] == 1


def test_backend_choice():
    assert D.pick_backend(8, 8) == "nccl"
    assert D.pick_backend(2, 1) == "gloo"


class _HostCounter:
    """The shared counter's host stand-in: a multiprocessing.Value (rank 0 resets it)."""

    def __init__(self, value, lock):
        self.value, self.lock = value, lock
        self.ptr = None

    def reset(self):
        with self.lock:
            self.value.value = 0


class _R:
    def __init__(self, count, h):
        self.count, self.hash = count, h


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_root, value, lock, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctr = _HostCounter(value, lock)
    loop = D.RankLoop(ctr, rank, world, "cpu")
    steps = []
    for _ in range(3):  # the counter is reset by rank 0 at every step
        info = {}

        def run(_ptr):
            c, h, chunks, taken = D.run_rank_cpu_standin(len(per_root), world, ctr.value, per_root, lock)
            info.update(chunks=chunks, taken=taken)
            return _R(c, h)

        c, h, r = loop.step(run)
        steps.append((c, h, r.count, info["chunks"], info["taken"]))
        dist.barrier()
    out[rank] = (steps, D.max_over_ranks(float(rank + 1) * 1.5, "cpu"))
    dist.destroy_process_group()


def test_gloo_world2_rank_loop_shared_counter():
    import oracle
    from paper_2401_05039_b200 import inputs as I

    g = I.erdos_renyi_c1b()
    tot = oracle.mbea(g)
    deg = np.bincount(g.col_idx, minlength=g.n2)
    roots = np.nonzero(deg > 0)[0]
    pr = oracle.mbea_roots(g, roots, candidate_side=2)
    per_root = [(int(a), int(b)) for a, b in pr[:, :2]]
    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    value = ctx.Value("q", 0, lock=False)
    lock = ctx.Lock()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_root, value, lock, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    for k in range(3):
        taken = []
        for r in range(world):
            steps, mx = out[r]
            c, h, own, chunks, t = steps[k]
            assert (c, h) == (tot.count, tot.hash)  # the all-reduce of the shares is the whole
            assert mx == 3.0
            taken += t
        assert sorted(taken) == list(range(len(roots)))  # every level-1 subtree claimed exactly once
    shares = [out[r][0][0][2] for r in range(world)]
    assert sum(shares) == tot.count
