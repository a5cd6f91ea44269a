"""Multi-GPU driver: one process per GPU, level-1 subtrees claimed through one shared counter.

The work shards with no data-path collective (level-1 subtrees are independent,
P:344-347): every rank runs the whole search kernel on its own GPU over the level-1 subtrees it
claims, in guided-self-scheduling chunks, from ONE counter that lives in rank 0's device memory and
is shared through a CUDA IPC handle (include/mbe.h mbe_counter_*).  The only collective is the final
all-reduce of (count, hash) — over NCCL when every rank has its own GPU, over gloo when several
ranks share one (NCCL refuses duplicate GPUs; the payload is 64 bytes either way).

Host logic only (argument marshalling, process-group plumbing): every step of the search runs in
libmbe's kernels.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from typing import Callable, List, Optional, Tuple

MASK64 = (1 << 64) - 1


# ------------------------------------------------------------------ guided self-scheduling
def gss_chunk(remaining: int, world: int) -> int:
    """Chunk size the kernel claims from the shared counter (search.cu claim_root_shared):
    ceil(remaining / (4 * world)), at least 1."""
    return max(1, -(-remaining // (4 * world)))


def gss_schedule(n_roots: int, world: int) -> List[Tuple[int, int]]:
    """The sequence of (start, length) chunks the shared counter hands out, in claim order."""
    out, pos = [], 0
    while pos < n_roots:
        c = min(gss_chunk(n_roots - pos, world), n_roots - pos)
        out.append((pos, c))
        pos += c
    return out


# ------------------------------------------------------------------ environment / process group
def dist_env() -> Tuple[int, int, int]:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def pick_backend(world: int, n_devices: int) -> str:
    """NCCL when every rank has its own GPU; gloo when ranks share GPUs (NCCL rejects duplicates)."""
    return "nccl" if n_devices >= world else "gloo"


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(world: int, argv: List[str]) -> int:
    """Launch `world` copies of this program as ranks 0..world-1 on 127.0.0.1 (what torchrun does),
    wait for all of them, and return the first nonzero exit code (0 if all succeeded)."""
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(world), LOCAL_WORLD_SIZE=str(world),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable] + argv, env=env))
    rc = 0
    for p in procs:
        c = p.wait()
        rc = rc or c
    return rc


# ------------------------------------------------------------------ the one collective
def limbs_of(count: int, h: int) -> List[int]:
    """(count, hash) -> 8 int64 limbs of 16 bits, so a sum over <= 2^47 ranks cannot overflow."""
    out = []
    for v in (count & MASK64, h & MASK64):
        out += [(v >> (16 * k)) & 0xFFFF for k in range(4)]
    return out


def from_limbs(limbs) -> Tuple[int, int]:
    vals = []
    for j in range(2):
        v = 0
        for k in range(4):
            v += int(limbs[4 * j + k]) << (16 * k)
        vals.append(v & MASK64)
    return vals[0], vals[1]


def allreduce_result(count: int, h: int, device, group=None) -> Tuple[int, int]:
    """Sum (count, hash mod 2^64) over ranks: the only data collective of the path."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(limbs_of(count, h), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return from_limbs(t.tolist())


def max_over_ranks(x: float, device, group=None) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_floats(x: float, device, world: int, group=None) -> List[float]:
    import torch
    import torch.distributed as dist

    t = torch.zeros(world, dtype=torch.float64, device=device)
    t[int(dist.get_rank(group))] = x
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [float(v) for v in t.tolist()]


# ------------------------------------------------------------------ shared counter
def share_counter(device: int, rank: int, make: Callable, open_: Callable, group=None):
    """Rank 0 creates the counter (``make(device)``) and broadcasts its 64-byte IPC handle; the other
    ranks open it (``open_(device, handle)``).  Returns this rank's counter object."""
    import torch.distributed as dist

    obj = [None]
    ctr = None
    if rank == 0:
        ctr = make(device)
        obj[0] = ctr.ipc_handle()
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank != 0:
        ctr = open_(device, obj[0])
    return ctr


class RankLoop:
    """One rank's step: (rank 0) zero the shared counter -> barrier -> run this rank's claims ->
    all-reduce (count, hash).  ``run(claim_counter)`` does the rank's enumeration and returns an object
    with .count and .hash (libmbe's Result on a GPU)."""

    def __init__(self, counter, rank: int, world: int, reduce_device, group=None):
        self.counter, self.rank, self.world, self.dev, self.group = counter, rank, world, reduce_device, group

    def step(self, run: Callable) -> Tuple[int, int, object]:
        import torch.distributed as dist

        if self.rank == 0:
            self.counter.reset()
        dist.barrier(group=self.group)
        r = run(self.counter.ptr)
        c, h = allreduce_result(r.count, r.hash, self.dev, self.group) if self.world > 1 else (r.count, r.hash)
        return c, h, r


def run_rank_cpu_standin(n_roots: int, world: int, counter, per_root, lock) -> Tuple[int, int, int, List[int]]:
    """Host stand-in of the kernel's claim protocol for CPU tests: draw chunks from a shared counter
    exactly as claim_root_shared does (one atomic add of gss_chunk per chunk) and sum the given per-root
    (count, hash) results of the claimed positions.  Returns (count, hash, chunks, positions)."""
    count = h = chunks = 0
    taken = []
    while True:
        with lock:
            g0 = counter.value
            if g0 >= n_roots:
                break
            c = gss_chunk(n_roots - g0, world)
            pos = counter.value
            counter.value = pos + c
        if pos >= n_roots:
            break
        chunks += 1
        for k in range(pos, min(pos + c, n_roots)):
            taken.append(k)
            count += int(per_root[k][0])
            h = (h + int(per_root[k][1])) & MASK64
    return count, h, chunks, taken
