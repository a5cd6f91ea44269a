"""Pins of the CPU oracle against what the paper and the mathematics fix.

No GPU, no product code: only oracle/ and the shared input generator.  Each
pin is chosen so that a plausible oracle bug fails it:
  * hash constants / rotation / size terms  -> splitmix64 vectors, closed-form hashes
  * a dropped maximality check or wrong P'/Q' threshold (Z3) -> brute force, crown 2^n-2
  * empty-side emission (Z1) -> isolated-vertex and brute-force comparisons
  * orientation / relabel mistakes -> side swap + candidate side metamorphic tests
  * wrong root-restriction shortcut -> plain literal MBEA gives the same tree
"""
import os

import numpy as np
import pytest

import oracle
from oracle import reference as R
from paper_2401_05039_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def spec_path():
    """SPEC S:283 path: rows a0,a1; cols b0,b1; edges a0b0, a0b1, a1b1."""
    return I.from_edges(2, 2, [0, 0, 1], [0, 1, 1], name="spec_path")


def _closed_form_graph(name):
    if name.startswith("crown"):
        return I.crown(int(name[5:]))
    if name.startswith("match"):
        return I.perfect_matching(int(name[5:]))
    if name == "spec_path":
        return spec_path()
    m, n = name[1:].split(",")
    return I.complete(int(m), int(n))


# ------------------------------------------------------------------ mix64
def test_mix64_published_splitmix64_vectors():
    G = 0x9E3779B97F4A7C15
    for k, v in _read_golden("splitmix64_seed0.txt"):
        z = (int(k) * G) & R.MASK64
        assert R.mix64(z) == int(v, 16)
        assert oracle.mix64(z) == int(v, 16)


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("row", _read_golden("closed_forms.txt"), ids=lambda r: r[0])
def test_closed_form_golden(row):
    name, count, h = row[0], int(row[1]), int(row[2], 16)
    g = _closed_form_graph(name)
    r = oracle.mbea(g, check=True)
    assert (r.count, r.hash, r.bad) == (count, h, 0)


@pytest.mark.parametrize("n", [2, 3, 4, 6, 8, 10, 12])
def test_crown_closed_form(n):
    # M(S_n) = {(S, [n] \ S) : ∅ ≠ S ⊊ [n]}  ->  2^n - 2 bicliques
    fam = []
    for S in range(1, (1 << n) - 1):
        A = tuple(i for i in range(n) if S >> i & 1)
        B = tuple(j for j in range(n) if not S >> j & 1)
        fam.append((A, B))
    g = I.crown(n)
    r = oracle.mbea(g)
    assert r.count == (1 << n) - 2
    assert r.hash == R.result_hash(fam)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 7), (3, 5), (6, 2), (9, 9)])
def test_complete_closed_form(m, n):
    g = I.complete(m, n)
    r = oracle.mbea(g)
    assert r.count == 1
    assert r.hash == R.biclique_hash(tuple(range(m)), tuple(range(n)))


@pytest.mark.parametrize("n", [1, 5, 17])
def test_matching_closed_form(n):
    r = oracle.mbea(I.perfect_matching(n))
    assert r.count == n
    assert r.hash == R.result_hash([((i,), (i,)) for i in range(n)])


@pytest.mark.parametrize("m", [3, 4, 5, 8, 13])
def test_path_closed_form(m):
    # a path with m vertices has m-2 maximal bicliques (the stars of its inner vertices)
    assert oracle.mbea(I.path(m)).count == m - 2


def test_disjoint_blocks_and_star():
    g = I.disjoint_blocks([(2, 3), (1, 1), (4, 2), (3, 3)])
    assert oracle.mbea(g).count == 4
    s = I.star(6)
    r = oracle.mbea(s)
    assert r.count == 1 and r.hash == R.biclique_hash((0,), tuple(range(6)))


def test_empty_graphs():
    for n1, n2 in [(0, 0), (0, 5), (4, 0), (5, 7)]:
        g = I.from_edges(n1, n2, [], [])
        r = oracle.mbea(g)
        assert (r.count, r.hash, r.tasks) == (0, 0, 0)


# ------------------------------------------------------------------ brute force
def _random_graphs(n_graphs, max_side, seed0):
    ps = [0.1, 0.3, 0.5, 0.7, 0.9]
    for k in range(n_graphs):
        z = R.mix64(seed0 + k)
        n1 = 1 + z % max_side
        n2 = 1 + (z >> 8) % max_side
        yield I.random_bipartite(n1, n2, ps[k % 5], seed0 * 1000 + k)


def test_oracle_equals_closure_bruteforce_1000_graphs():
    """>= 1,000 random graphs, sides <= 10, p in 0.1-0.9, fixed seeds."""
    for g in _random_graphs(1000, 10, 11):
        truth = R.maximal_bicliques_closure(g)
        lst = oracle.mbea_list(g)
        assert len(lst) == len(set(lst)), "duplicate emission"
        assert set(lst) == truth
        r = oracle.mbea(g, threads=2, check=True)
        assert r.count == len(truth)
        assert r.hash == R.result_hash(truth)
        assert r.bad == 0


def test_oracle_orders_and_sides_agree_with_bruteforce():
    for g in _random_graphs(300, 12, 23):
        truth = R.maximal_bicliques_closure(g)
        h = R.result_hash(truth)
        for side in (1, 2):
            for order in ("ascending", "input"):
                r = oracle.mbea(g, candidate_side=side, order=order)
                assert (r.count, r.hash) == (len(truth), h)


def test_next_closure_equals_closure_bruteforce():
    for g in _random_graphs(200, 9, 37):
        assert R.maximal_bicliques_next_closure(g) == R.maximal_bicliques_closure(g)


def test_plain_literal_mbea_same_tree_as_root_shortcut():
    """The root 2-hop restriction is exact: same result AND same search tree."""
    for g in list(_random_graphs(100, 14, 41)) + [I.crown(8), I.erdos_renyi_c1b(60, 60)]:
        a = oracle.mbea(g)
        b = oracle.mbea_plain(g)
        assert (a.count, a.hash, a.tasks, a.pruned) == (b.count, b.hash, b.tasks, b.pruned)
        assert b.bad == 0


# ------------------------------------------------------------------ C1b golden
def test_c1b_golden_next_closure_and_mbea():
    gold = {k: v for k, v in _read_golden("c1b_er200.txt")}
    g = I.erdos_renyi_c1b()
    assert g.n_edges == int(gold["edges"])
    nc = R.maximal_bicliques_next_closure(g)
    assert len(nc) == int(gold["count"])
    assert R.result_hash(nc) == int(gold["hash"], 16)
    for side in (1, 2):
        r = oracle.mbea(g, candidate_side=side, check=True)
        assert (r.count, r.hash, r.bad) == (int(gold["count"]), int(gold["hash"], 16), 0)


# ------------------------------------------------------------------ metamorphic
def test_metamorphic_swap_isolated_duplicates_permutation():
    g = I.erdos_renyi_c1b(80, 50)
    base = oracle.mbea(g)
    # swap sides: hash of the transposed set = hash with A/B roles swapped
    gt = g.transpose()
    lst = oracle.mbea_list(g)
    swapped = [(B, A) for A, B in lst]
    assert oracle.mbea(gt).hash == R.result_hash(swapped)
    assert oracle.mbea(gt).count == base.count
    # isolated vertices appended on both sides
    e = g.edges()
    gi = I.from_edges(g.n1 + 7, g.n2 + 3, e[:, 0], e[:, 1])
    assert (oracle.mbea(gi).count, oracle.mbea(gi).hash) == (base.count, base.hash)
    # duplicate edges (not deduplicated in the CSR): same result
    gd = I.from_edges(g.n1, g.n2, np.concatenate([e[:, 0], e[:40, 0]]), np.concatenate([e[:, 1], e[:40, 1]]),
                      dedup=False)
    assert gd.n_edges == g.n_edges + 40
    assert (oracle.mbea(gd).count, oracle.mbea(gd).hash) == (base.count, base.hash)
    # permuted ids: map the listing back
    rng = np.random.default_rng(5)
    p1 = rng.permutation(g.n1)
    p2 = rng.permutation(g.n2)
    gp = I.from_edges(g.n1, g.n2, p1[e[:, 0]], p2[e[:, 1]])
    mapped = {(tuple(sorted(int(p1[a]) for a in A)), tuple(sorted(int(p2[b]) for b in B))) for A, B in lst}
    assert set(oracle.mbea_list(gp)) == mapped


def test_per_root_sums_equal_total():
    g = I.erdos_renyi_c1b()
    for side in (1, 2):
        tot = oracle.mbea(g, candidate_side=side)
        n = g.n1 if side == 1 else g.n2
        pr = oracle.mbea_roots(g, np.arange(n), candidate_side=side)
        assert int(pr[:, 0].sum()) == tot.count
        assert int(pr[:, 1].astype(object).sum()) & R.MASK64 == tot.hash
        assert int(pr[:, 2].sum()) == tot.tasks
        assert int(pr[:, 3].sum()) == tot.pruned


def test_invalid_input_rejected():
    g = I.from_edges(2, 2, [0, 1], [0, 1])
    bad = I.Graph(2, 2, g.row_ptr, np.array([0, 5], dtype=np.uint32))
    with pytest.raises(ValueError):
        oracle.mbea(bad)
    bad2 = I.Graph(2, 2, np.array([0, 2, 1], dtype=np.uint64), np.array([0, 1], dtype=np.uint32))
    with pytest.raises(ValueError):
        oracle.mbea(bad2)


# ------------------------------------------------------------------ listing text
def test_listing_text_worked_example():
    """SPEC.md S:544 ("DESIGN DECISIONS"): `L: id,... | R: id,...`, original ids, lines sorted
    lexicographically (bytewise: "L: 1 " < "L: 10" < "L: 2").  Bicliques worked out by hand:
    rows 0:{0,1}, 1:{1,2}, 2:{10}, 10:{5} -> ({0},{0,1}), ({0,1},{1}), ({1},{1,2}), ({10},{5}), ({2},{10})."""
    g = I.from_edges(11, 11, [0, 0, 1, 1, 2, 10], [0, 1, 1, 2, 10, 5])
    want = (b"L: 0 | R: 0,1\n"
            b"L: 0,1 | R: 1\n"
            b"L: 1 | R: 1,2\n"
            b"L: 10 | R: 5\n"
            b"L: 2 | R: 10\n")
    assert R.listing_text(oracle.mbea_list(g)) == want
    assert R.listing_text(R.maximal_bicliques_closure(g)) == want
    assert R.listing_text([]) == b""


# ------------------------------------------------------------------ search-tree counters (tasks / pruned)
# A task is one popped candidate x with L' = L ∩ N(x) ≠ ∅ (Algorithm 1 Steps 1-2); it is
# pruned when Step 3 finds a Q vertex v with |N(v) ∩ L'| = |L'|.  Every candidate is
# retired into Q after its iteration, and P' is ordered by ascending (|N(v) ∩ L'|, r(v)),
# r = rank in the root order by (degree, original id) (reading Z6).  The
# values below are derived by hand from those rules alone, so a flipped sort, a tie-break on the
# original id instead of r(v), or a missing retirement of x into Q fails one of them.

@pytest.mark.parametrize("m,n", [(1, 1), (1, 7), (3, 5), (6, 2), (9, 9)])
def test_tree_complete(m, n):
    # K_{m,n}: candidates U_c = the smaller side (side 1 on a tie), all with N = V_c.  Root task 1:
    # L' = V_c, Q = ∅, every other candidate has c = |L'| -> R', so P' = ∅.  Every later root task
    # has the earlier candidates in Q with c = |L'| -> pruned.  (tasks, pruned) = (|U_c|, |U_c| - 1).
    k = min(m, n)
    r = oracle.mbea(I.complete(m, n))
    assert (r.count, r.tasks, r.pruned) == (1, k, k - 1)


@pytest.mark.parametrize("n", [1, 5, 17])
def test_tree_matching(n):
    # perfect matching: each root x has L' = {x's partner}, no other vertex meets it: n tasks, 0 pruned
    r = oracle.mbea(I.perfect_matching(n))
    assert (r.count, r.tasks, r.pruned) == (n, n, 0)


def test_tree_star():
    # star(6): one row joined to 6 cols; the row side (1 vertex) is the candidate side: one task
    r = oracle.mbea(I.star(6))
    assert (r.count, r.tasks, r.pruned) == (1, 1, 0)


def test_tree_crown3():
    # S_3, rows are candidates (tie -> side 1), N(0)={1,2}, N(1)={0,2}, N(2)={0,1}; all degree 2, so
    # the root order is 0,1,2.
    #  x=0: L'={1,2}, Q=∅; c(1)=|{2}|=1, c(2)=|{1}|=1 -> P'=[1,2]                     task 1
    #     x=1: L''={2}; c(2)=0                                                       task 2
    #     x=2: L''={1}; Q=[1]: c=0                                                   task 3
    #  x=1: L'={0,2}; Q=[0]: c=1 -> Q'; c(2)=1 -> P'=[2]                             task 4
    #     x=2: L''={0}; Q=[0]: c=0                                                   task 5
    #  x=2: L'={0,1}; Q=[0,1]: c=1, c=1 -> Q'; P=∅                                   task 6
    # 6 tasks, none pruned, 6 = 2^3 - 2 bicliques.
    r = oracle.mbea(I.crown(3))
    assert (r.count, r.tasks, r.pruned) == (6, 6, 0)


def nested_pair():
    """rows 0:{0,1,2}, 1:{0} (rows = candidates): the root order is by ascending degree."""
    return I.from_edges(2, 3, [0, 0, 0, 1], [0, 1, 2, 0], name="nested_pair")


def test_tree_root_order_ascending():
    # r(1) = 0 (degree 1), r(0) = 1 (degree 3): root order [1, 0].
    #  x=1: L'={0}, Q=∅; c(0)=1=|L'| -> R'; P'=∅                                      task 1
    #  x=0: L'={0,1,2}; Q=[1]: c=1 < 3 -> Q'; P=∅                                      task 2
    # (2, 0).  A descending root order gives x=0 first (P'=[1], one child task) and then x=1 pruned
    # by Q=[0]: (3, 1).
    r = oracle.mbea(nested_pair())
    assert (r.count, r.tasks, r.pruned) == (2, 2, 0)


def deep_order_graph():
    """rows 0:{1,2,4}, 1:{0,2,3}, 2:{2,3,4}; 5 cols; rows are candidates (3 < 5)."""
    return I.from_edges(3, 5, [0, 0, 0, 1, 1, 1, 2, 2, 2], [1, 2, 4, 0, 2, 3, 2, 3, 4], name="deep_order")


def test_tree_deep_order_ascending():
    # All degrees 3: root order 0,1,2 and r(v) = v.
    #  x=0: L'={1,2,4}; c(1)=|{2}|=1, c(2)=|{2,4}|=2 -> P' ascending = [1, 2]         task 1
    #     x=1: L''={2}; c(2)=1=|L''| -> R''                                           task 2
    #     x=2: L''={2,4}; Q=[1]: c=1 < 2 -> Q'                                         task 3
    #  x=1: L'={0,2,3}; Q=[0]: c=1 -> Q'; c(2)=|{2,3}|=2 -> P'=[2]                    task 4
    #     x=2: L''={2,3}; Q=[0]: c=1 < 2                                               task 5
    #  x=2: L'={2,3,4}; Q=[0,1]: c=2, c=2 < 3                                          task 6
    # (6, 0).  A DESCENDING child order runs x=2 before x=1 under x=0: x=2 gets L''={2,4} and a
    # child (x=1, L'''={2}), then x=1 (L''={2}) is pruned by Q=[2] (c=1=|L''|): (7, 1).
    r = oracle.mbea(deep_order_graph())
    assert (r.count, r.tasks, r.pruned) == (6, 6, 0)


def tie_break_graph():
    """rows 0:{0,1}, 1:{0,1,2}, 2:{0,1,3,4}, 3:{1,2,4}; 5 cols; rows are candidates (4 < 5)."""
    return I.from_edges(4, 5, [0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3], [0, 1, 0, 1, 2, 0, 1, 3, 4, 1, 2, 4],
                        name="tie_break")


def test_tree_tie_break_by_rank():
    # degrees 2,3,4,3 -> r(0)=0, r(1)=1, r(3)=2, r(2)=3; root order [0, 1, 3, 2].
    #  x=0: L'={0,1}; c(1)=2, c(2)=2 -> R'; c(3)=|{1}|=1 -> P'=[3]                     task 1
    #     x=3: L''={1}                                                                 task 2
    #  x=1: L'={0,1,2}; Q=[0]: c=2 < 3 -> Q'; c(3)=|{1,2}|=2, c(2)=|{0,1}|=2 -> P'
    #       keys tie at 2: r(3)=2 < r(2)=3 -> P'=[3, 2]                                 task 3
    #     x=3: L''={1,2}; Q=[0]: c=1 -> Q'; c(2)=|{1}|=1 -> P'=[2]                      task 4
    #        x=2: L'''={1}; Q=[0]: c=1=|L'''| -> pruned                                task 5 (pruned)
    #     x=2: L''={0,1}; Q=[0,3]: c(0)=2=|L''| -> pruned                              task 6 (pruned)
    #  x=3: L'={1,2,4}; Q=[0,1]: c=1, c=2 -> Q'; c(2)=|{1,4}|=2 -> P'=[2]              task 7
    #     x=2: L''={1,4}; Q=[0,1]: c=1, c=1                                            task 8
    #  x=2: L'={0,1,3,4}; Q=[0,1,3]: c=2,2,2 < 4                                       task 9
    # (9, 2), 7 bicliques.  Breaking the tie by ORIGINAL id instead ([2, 3] under x=1) gives
    # x=2 pruned at once (c(0)=2=|{0,1}|) and x=3 unpruned: (8, 1).
    r = oracle.mbea(tie_break_graph())
    assert (r.count, r.tasks, r.pruned) == (7, 9, 2)


def test_tree_counters_literal_mbea_agrees_on_worked_graphs():
    """The literal sequential MBEA(V, ∅, P, ∅) (no root shortcut) builds the same hand-derived trees."""
    for g, want in [(nested_pair(), (2, 2, 0)), (deep_order_graph(), (6, 6, 0)), (tie_break_graph(), (7, 9, 2)),
                    (I.crown(3), (6, 6, 0))]:
        b = oracle.mbea_plain(g)
        assert (b.count, b.tasks, b.pruned) == want, g.name


def test_tree_order_variants_hand_derived():
    """SURVEY §8(f) row 3 order ablations.  Descending: root P by (-deg, id), P' by (-|N(v) ∩ L'|, r(v));
    input: root P by id, P' in its parent's order.  Derivations in the comments of the tests above:
    nested_pair descending/input = x=0 first (child x=1), then x=1 pruned by Q=[0] -> (3, 1);
    deep_order descending -> (7, 1) (x=2 before x=1 under x=0); deep_order input keeps [1, 2] -> (6, 0)."""
    for g, order, want in [(nested_pair(), "descending", (2, 3, 1)), (nested_pair(), "input", (2, 3, 1)),
                           (deep_order_graph(), "descending", (6, 7, 1)), (deep_order_graph(), "input", (6, 6, 0))]:
        r = oracle.mbea(g, order=order)
        assert (r.count, r.tasks, r.pruned) == want, (g.name, order)
        b = oracle.mbea_plain(g, order=order)
        assert (b.count, b.tasks, b.pruned) == want, (g.name, order)


def test_descending_order_equals_bruteforce():
    for g in _random_graphs(200, 11, 59):
        truth = R.maximal_bicliques_closure(g)
        for side in (1, 2):
            r = oracle.mbea(g, candidate_side=side, order="descending")
            assert (r.count, r.hash) == (len(truth), R.result_hash(truth))
