"""Seeded synthetic bipartite inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no intersections, counts,
hashes of bicliques).  It only draws graphs.  Both sides of every parity test
receive the same arrays from here; neither side imports the other.

Every random number is counter-based: ``u64(seed, stream, index) =
splitmix64_finalizer(seed ^ (stream << 40) ^ index)``, so the output is a pure
function of the parameters (independent of thread count, batch size and
platform).  Graphs are returned as a row-CSR over ORIGINAL 0-based ids in the
input orientation: side 1 = rows (``n1``), side 2 = cols (``n2``) — the layout
``mbe_load_csr`` takes (include/mbe.h).

Configs (BASELINE.json ``configs``):
  C1a crown K_{12,12} minus a perfect matching, C1b G(200,200,0.05),
  C2..C5 power-law bipartite graphs shaped like the paper's KONECT datasets
  (Table 1: YouTube 94,238 x 30,087 / 293,360 E;
  stackoverflow 545,195 x 96,678 / 1,301,942 E; BookCrossing
  340,523 x 105,278 / 1,149,739 E; GitHub ~56,519 x 120,867 / ~440,237 E).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _rng_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based RNG: splitmix64 finalizer of seed ^ (stream<<40) ^ idx.

    This is the generator's own copy; the oracle and the CUDA path each keep a
    separate implementation of the (unrelated) biclique hash.
    """
    z = np.asarray(idx, dtype=np.uint64) ^ np.uint64((seed ^ (stream << 40)) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _uniform(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Uniform doubles in [0,1) with 53 random bits."""
    return (_rng_u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


@dataclasses.dataclass
class Graph:
    """Row-CSR over original ids: row i (side 1) -> cols (side 2)."""

    n1: int
    n2: int
    row_ptr: np.ndarray  # uint64 [n1+1]
    col_idx: np.ndarray  # uint32 [nnz]
    name: str = ""
    params: Optional[dict] = None

    @property
    def n_edges(self) -> int:
        return int(self.row_ptr[-1])

    def edges(self) -> np.ndarray:
        """(nnz, 2) array of (row, col)."""
        rows = np.repeat(np.arange(self.n1, dtype=np.uint32), np.diff(self.row_ptr).astype(np.int64))
        return np.stack([rows, self.col_idx.astype(np.uint32)], axis=1)

    def transpose(self) -> "Graph":
        """Same edge set with the sides swapped (a metamorphic test input)."""
        e = self.edges()
        return from_edges(self.n2, self.n1, e[:, 1], e[:, 0], name=self.name + "^T")


def from_edges(n1: int, n2: int, rows, cols, name: str = "", params: Optional[dict] = None,
               dedup: bool = True) -> Graph:
    """Row-CSR from an edge list (rows sorted; optional dedup)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if rows.size:
        key = rows * max(n2, 1) + cols
        if dedup:
            key = np.unique(key)
        else:
            key = np.sort(key)
        rows = key // max(n2, 1)
        cols = key % max(n2, 1)
    counts = np.bincount(rows, minlength=n1) if n1 else np.zeros(0, dtype=np.int64)
    row_ptr = np.zeros(n1 + 1, dtype=np.uint64)
    if n1:
        row_ptr[1:] = np.cumsum(counts).astype(np.uint64)
    return Graph(n1, n2, row_ptr, cols.astype(np.uint32), name=name, params=params)


# ---------------------------------------------------------------- closed forms
def crown(n: int) -> Graph:
    """Crown graph S_n = K_{n,n} minus a perfect matching: edge (i,j) iff i != j."""
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    m = i != j
    return from_edges(n, n, i[m], j[m], name=f"crown{n}")


def complete(m: int, n: int) -> Graph:
    i, j = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    return from_edges(m, n, i.ravel(), j.ravel(), name=f"K{m},{n}")


def perfect_matching(n: int) -> Graph:
    return from_edges(n, n, np.arange(n), np.arange(n), name=f"match{n}")


def path(m: int) -> Graph:
    """Path with m vertices a0-b0-a1-b1-... (alternating sides)."""
    rows, cols = [], []
    for k in range(m - 1):
        # vertex k: side 1 if k even (id k//2), side 2 if odd (id k//2)
        if k % 2 == 0:
            rows.append(k // 2)
            cols.append(k // 2)
        else:
            rows.append((k + 1) // 2)
            cols.append(k // 2)
    n1 = (m + 1) // 2
    n2 = m // 2
    return from_edges(n1, n2, rows, cols, name=f"path{m}")


def disjoint_blocks(sizes) -> Graph:
    """Disjoint union of complete blocks K_{a,b}."""
    rows, cols = [], []
    o1 = o2 = 0
    for a, b in sizes:
        i, j = np.meshgrid(np.arange(a), np.arange(b), indexing="ij")
        rows.append(i.ravel() + o1)
        cols.append(j.ravel() + o2)
        o1 += a
        o2 += b
    return from_edges(o1, o2, np.concatenate(rows) if rows else [], np.concatenate(cols) if cols else [],
                      name="blocks")


def star(k: int) -> Graph:
    return from_edges(1, k, np.zeros(k, dtype=np.int64), np.arange(k), name=f"star{k}")


# ---------------------------------------------------------------- random graphs
C1B_SEED = 0x2401050390000001
C1B_THRESHOLD = 922337203685477580  # floor(2^64 / 20): p = 0.05 as an exact integer compare


def erdos_renyi_c1b(n1: int = 200, n2: int = 200, seed: int = C1B_SEED,
                    threshold: int = C1B_THRESHOLD) -> Graph:
    """edge (i,j) iff mix64(seed ^ (i*n2+j)) < threshold (integer compare)."""
    i, j = np.meshgrid(np.arange(n1, dtype=np.uint64), np.arange(n2, dtype=np.uint64), indexing="ij")
    idx = (i * np.uint64(n2) + j).ravel()
    z = _rng_u64(seed, 0, idx)
    m = z < np.uint64(threshold)
    return from_edges(n1, n2, i.ravel()[m].astype(np.int64), j.ravel()[m].astype(np.int64),
                      name=f"er{n1}x{n2}", params={"seed": seed, "threshold": threshold})


def random_bipartite(n1: int, n2: int, p: float, seed: int) -> Graph:
    """Small Erdos-Renyi bipartite graph (tests)."""
    if n1 == 0 or n2 == 0:
        return from_edges(n1, n2, [], [])
    i, j = np.meshgrid(np.arange(n1, dtype=np.uint64), np.arange(n2, dtype=np.uint64), indexing="ij")
    idx = (i * np.uint64(n2) + j).ravel()
    u = _uniform(seed, 7, idx)
    m = u < p
    return from_edges(n1, n2, i.ravel()[m].astype(np.int64), j.ravel()[m].astype(np.int64),
                      name=f"rnd{n1}x{n2}p{p}s{seed}")


# ---------------------------------------------------------------- power-law (Chung-Lu)
def _weighted_sampler(weights: np.ndarray):
    cdf = np.cumsum(weights)
    cdf /= cdf[-1]

    def draw(u: np.ndarray) -> np.ndarray:
        return np.minimum(np.searchsorted(cdf, u, side="right"), len(cdf) - 1).astype(np.int64)

    return draw


def power_law(n1: int, n2: int, n_edges: int, seed: int, gamma1: float, gamma2: float,
              i0_1: float = 1.0, i0_2: float = 1.0, blocks: int = 0, block_a: int = 30,
              block_b: int = 15, block_p: float = 0.7, block_uniform: bool = False, name: str = "") -> Graph:
    """Bipartite Chung-Lu with min degree 1 on both sides (SURVEY §8(d) recipe).

    * side-s weight of rank i: (i + i0_s)^(-1/(gamma_s - 1)); ranks are mapped to
      ids through a seeded permutation, so id order != degree order;
    * min degree 1: every vertex of the larger side gets one edge to a
      weight-drawn vertex of the other side, then every still-isolated vertex of
      the smaller side gets one edge to a weight-drawn vertex of the larger side;
    * optional planted communities: ``blocks`` overlapping a x b blocks whose
      members are drawn by weight (or uniformly with ``block_uniform``), each
      pair an edge with prob ``block_p``;
    * then Chung-Lu pairs (both endpoints weight-drawn) until exactly
      ``n_edges`` distinct edges (first occurrences in counter order).
    """
    params = dict(n1=n1, n2=n2, n_edges=n_edges, seed=seed, gamma1=gamma1, gamma2=gamma2,
                  i0_1=i0_1, i0_2=i0_2, blocks=blocks, block_a=block_a, block_b=block_b,
                  block_p=block_p, block_uniform=block_uniform)
    # rank -> id permutations
    perm1 = np.argsort(_rng_u64(seed, 1, np.arange(n1)), kind="stable")
    perm2 = np.argsort(_rng_u64(seed, 2, np.arange(n2)), kind="stable")
    w1 = np.empty(n1)
    w2 = np.empty(n2)
    w1[perm1] = (np.arange(n1) + i0_1) ** (-1.0 / (gamma1 - 1.0))
    w2[perm2] = (np.arange(n2) + i0_2) ** (-1.0 / (gamma2 - 1.0))
    draw1 = _weighted_sampler(w1)
    draw2 = _weighted_sampler(w2)

    keys: list[np.ndarray] = []
    # 1) min degree 1
    if n1 >= n2:
        r = np.arange(n1, dtype=np.int64)
        c = draw2(_uniform(seed, 3, np.arange(n1)))
        keys.append(r * n2 + c)
        covered = np.zeros(n2, dtype=bool)
        covered[c] = True
        miss = np.nonzero(~covered)[0]
        r2 = draw1(_uniform(seed, 4, miss))
        keys.append(r2 * n2 + miss)
    else:
        c = np.arange(n2, dtype=np.int64)
        r = draw1(_uniform(seed, 3, np.arange(n2)))
        keys.append(r * n2 + c)
        covered = np.zeros(n1, dtype=bool)
        covered[r] = True
        miss = np.nonzero(~covered)[0]
        c2 = draw2(_uniform(seed, 4, miss))
        keys.append(miss * n2 + c2)
    # 2) planted communities
    for b in range(blocks):
        base = b * (block_a + block_b + block_a * block_b)
        ua = _uniform(seed, 5, base + np.arange(block_a))
        ub = _uniform(seed, 5, base + block_a + np.arange(block_b))
        if block_uniform:
            ra = np.minimum((ua * n1).astype(np.int64), n1 - 1)
            cb = np.minimum((ub * n2).astype(np.int64), n2 - 1)
        else:
            ra = draw1(ua)
            cb = draw2(ub)
        pu = _uniform(seed, 5, base + block_a + block_b + np.arange(block_a * block_b))
        ii, jj = np.meshgrid(ra, cb, indexing="ij")
        m = (pu < block_p).reshape(block_a, block_b)
        keys.append(ii[m] * n2 + jj[m])

    def first_unique(k: np.ndarray) -> np.ndarray:
        _, first = np.unique(k, return_index=True)
        return k[np.sort(first)]

    have = first_unique(np.concatenate(keys))
    if have.size > n_edges:
        raise ValueError(f"n_edges={n_edges} below the {have.size} edges forced by min-degree/blocks")
    # 3) Chung-Lu fill in counter order
    counter = 0
    batch = max(1 << 16, n_edges // 4)
    while have.size < n_edges:
        idx = np.arange(counter, counter + batch)
        counter += batch
        r = draw1(_uniform(seed, 8, idx))
        c = draw2(_uniform(seed, 9, idx))
        k = first_unique(r * n2 + c)
        k = k[~np.isin(k, have, assume_unique=True)]
        need = n_edges - have.size
        have = np.concatenate([have, k[:need]])
    rows = have // n2
    cols = have % n2
    return from_edges(n1, n2, rows, cols, name=name or f"pl{n1}x{n2}", params=params)


# ---------------------------------------------------------------- named configs
# Frozen generator parameters for the BASELINE.json configs.  Seeds follow the
# SURVEY's convention 0x24010503900000NN.  Shapes are the paper's Table 1
# sizes and BASELINE.json's GitHub shape.
CONFIGS = {
    "C2": dict(n1=94238, n2=30087, n_edges=293360, seed=0x2401050390000002,
               gamma1=2.5, gamma2=2.1, i0_1=1.0, i0_2=8.0, name="C2-youtube"),
    "C3": dict(n1=56519, n2=120867, n_edges=440237, seed=0x2401050390000003,
               gamma1=2.1, gamma2=2.5, i0_1=8.0, i0_2=1.0, name="C3-github"),
    "C4": dict(n1=105278, n2=340523, n_edges=1149739, seed=0x2401050390000004,
               gamma1=2.1, gamma2=2.5, i0_1=16.0, i0_2=1.0, name="C4-bookcrossing"),
    "C5": dict(n1=545195, n2=96678, n_edges=1301942, seed=0x2401050390000005,
               gamma1=2.5, gamma2=2.1, i0_1=1.0, i0_2=16.0, name="C5-stackoverflow"),
    # C5 with planted communities (SURVEY §8(d) "optional planted communities", §8(e) second scaling
    # point): the same vertex sets and generator, plus 3,000 overlapping 30 x 15 blocks at p = 0.7
    # (members drawn uniformly: weight-drawn members put every hub in hundreds of blocks and the
    # oracle did not finish a 0.5 % root sample in 40 min), which lifts nMB/|E| toward the paper's community-rich datasets
    # (P:627-630).  The blocks force ~1.5 M edges, so |E| is raised to 2,000,000.
    "C5p": dict(n1=545195, n2=96678, n_edges=2000000, seed=0x2401050390000015,
                gamma1=2.5, gamma2=2.1, i0_1=1.0, i0_2=16.0, blocks=3000, block_a=30, block_b=15,
                block_p=0.7, block_uniform=True, name="C5p-stackoverflow-planted"),
}


def config_graph(name: str) -> Graph:
    """The graph of a named config: C1a, C1b, C2..C5."""
    if name == "C1a":
        return crown(12)
    if name == "C1b":
        return erdos_renyi_c1b()
    if name in CONFIGS:
        return power_law(**CONFIGS[name])
    raise KeyError(name)
