"""Pure-Python definitions of the result (TEST INFRASTRUCTURE ONLY).

* ``maximal_bicliques_closure`` — the plain definition of: a biclique
  (A,B) is maximal iff no vertex can be added to either side, i.e. A = N(B)
  and B = N(A).  Enumerates every nonempty subset S of the smaller side and
  closes it: B = N(S), A = N(B) ("closure_enumerate").
* ``maximal_bicliques_next_closure`` — Ganter's Next-Closure (formal concept
  analysis, lectic order), an independent textbook enumeration of all closed
  pairs; concepts with an empty side are dropped (reading Z1).
* ``result_hash`` — the order-independent 64-bit result hash (DESIGN.md,
  SURVEY §8(c)): Σ H(A,B) mod 2^64 with
  H(A,B) = mix64(sA ^ rotl64(sB,32) ^ (|A|<<32) ^ |B|),
  sA = Σ mix64(2a), sB = Σ mix64(2b+1), a/b original 0-based ids of side 1/2.
* ``listing_text`` — the canonical listing text of SPEC.md S:544 ("DESIGN
  DECISIONS": one biclique per line, ``L: id,id,... | R: id,id,...`` with
  original ids, lines sorted lexicographically), ids ascending within a side.

Graphs are the row-CSR ``inputs.Graph`` objects (n1, n2, row_ptr, col_idx);
this module only reads those arrays.
"""
from __future__ import annotations

MASK64 = 0xFFFFFFFFFFFFFFFF


def mix64(z: int) -> int:
    """splitmix64 finalizer (Steele, Lea, Flood 2014; Vigna's splitmix64.c)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def rotl64(v: int, k: int) -> int:
    return ((v << k) | (v >> (64 - k))) & MASK64


def biclique_hash(A, B) -> int:
    sA = sum(mix64(2 * a) for a in A) & MASK64
    sB = sum(mix64(2 * b + 1) for b in B) & MASK64
    return mix64(sA ^ rotl64(sB, 32) ^ ((len(A) << 32) & MASK64) ^ len(B))


def result_hash(bicliques) -> int:
    return sum(biclique_hash(A, B) for A, B in bicliques) & MASK64


def listing_text(bicliques) -> bytes:
    """SPEC S:544 text: one line per (A, B), ids ascending per side, lines sorted bytewise."""
    lines = []
    for A, B in bicliques:
        lines.append(("L: " + ",".join(str(a) for a in sorted(A)) + " | R: "
                      + ",".join(str(b) for b in sorted(B)) + "\n").encode("ascii"))
    return b"".join(sorted(lines))


def _masks(g):
    rows = [0] * g.n1
    cols = [0] * g.n2
    rp = [int(v) for v in g.row_ptr]
    ci = [int(v) for v in g.col_idx]
    for i in range(g.n1):
        for e in range(rp[i], rp[i + 1]):
            j = ci[e]
            rows[i] |= 1 << j
            cols[j] |= 1 << i
    return rows, cols


def _bits(m: int):
    out = []
    k = 0
    while m:
        if m & 1:
            out.append(k)
        m >>= 1
        k += 1
    return tuple(out)


def maximal_bicliques_closure(g, limit: int = 20):
    """{(A, B)}: closures of every nonempty subset of the smaller side."""
    rows, cols = _masks(g)
    all1 = (1 << g.n1) - 1
    all2 = (1 << g.n2) - 1
    out = set()
    if g.n1 <= g.n2:
        if g.n1 > limit:
            raise ValueError("side too large for brute force")
        for S in range(1, 1 << g.n1):
            B = all2
            for i in _bits(S):
                B &= rows[i]
            if not B:
                continue
            A = all1
            for j in _bits(B):
                A &= cols[j]
            out.add((_bits(A), _bits(B)))
    else:
        if g.n2 > limit:
            raise ValueError("side too large for brute force")
        for S in range(1, 1 << g.n2):
            A = all1
            for j in _bits(S):
                A &= cols[j]
            if not A:
                continue
            B = all2
            for i in _bits(A):
                B &= rows[i]
            out.add((_bits(A), _bits(B)))
    return out


def maximal_bicliques_next_closure(g):
    """Ganter's Next-Closure over intents (attributes = side-2 ids)."""
    rows, cols = _masks(g)
    n2 = g.n2
    all1 = (1 << g.n1) - 1
    all2 = (1 << n2) - 1

    def extent(B: int) -> int:
        A = all1
        m = B
        j = 0
        while m:
            if m & 1:
                A &= cols[j]
            m >>= 1
            j += 1
        return A

    def intent(A: int) -> int:
        B = all2
        m = A
        i = 0
        while m:
            if m & 1:
                B &= rows[i]
            m >>= 1
            i += 1
        return B

    out = set()
    B = intent(extent(0))
    while True:
        A = extent(B)
        if A and B:
            out.add((_bits(A), _bits(B)))
        if B == all2:
            break
        nxt = None
        for i in range(n2 - 1, -1, -1):
            bit = 1 << i
            if B & bit:
                continue
            low = B & (bit - 1)
            C = intent(extent(low | bit))
            if (C & ~B) & (bit - 1) == 0:  # no new element below i
                nxt = C
                break
        if nxt is None:
            break
        B = nxt
    return out
