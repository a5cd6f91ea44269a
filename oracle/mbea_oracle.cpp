// oracle/mbea_oracle.cpp — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this library.  The product path
// (paper_2401_05039_b200/, libmbe.so) never links, imports or calls it, and it
// shares no code with it (no headers, no helpers, no tables).
//
// What it computes: the maximal bicliques of a bipartite graph, §II-A
// (P:87-98): (A,B) with A x B ⊆ E, A = N(B), B = N(A), both sides nonempty
// (reading Z1 of DESIGN.md), reported as
//     count = |M(G)|,
//     hash  = Σ H(A,B) mod 2^64.
//
// How: Algorithm 1 "MBEA(L,R,P,Q)" (prose P:179-201), written out
// step by step with plain std::vector set copies per level:
//   Step 1 candidate selection  x = P.pop(); R' = R ∪ {x}
//   Step 2 L' construction      L' = {v ∈ L : (x,v) ∈ E}
//   Step 3 maximality check     over Q, forward counts |N(v)∩L'|
//   Step 4 maximal expansion    over P, forward counts
//   recurse if P' ≠ ∅; Q = Q ∪ {x}
// Readings taken where the paper is silent or garbled:
//   Z1  L' = ∅ → skip x (no empty-side biclique); degree-0 vertices are not in
//       the root P.
//   Z2  L', P', Q' are reset every iteration (P:125 declares them once).
//   Z3  P' = {v : 0 < |N(v)∩L'| < |L'|} (Alg. 1 line P:157; P:523's "y>|L'|"
//       is a typo).
//   Z6  candidate order: iMBE ascending |N(v)∩L|; the
//       root P is ordered by (degree, original id) = rank r(v); every P' is
//       sorted by (|N(v)∩L'|, r(v)).  order_mode=1 pops in input order instead
//       (result-invariant; used to check order independence on small graphs).
//       order_mode=2 is the descending ablation: the root P
//       by (descending degree, original id), every P' by (descending
//       |N(v)∩L'|, r(v)), r = position in that root order.
// One exact shortcut (result-identical): at the root, L = V, so a
// vertex v with N(v)∩N(x) = ∅ has count 0 and Algorithm 1 ignores it (it
// cannot break maximality since |L'| > 0 and joins neither Q' nor P').  The
// root iteration for x therefore scans only v ∈ N(N(x)), in the root order.
// Root iterations are independent given their position i in the root order
// (Q = P[0..i-1], P = P[i+1..], exactly what the sequential loop holds), so
// they run on std::thread workers; everything below level 1 is serial.
//
// No compact arrays, no reverse scanning, no bitmaps, no relabelling: vertices
// keep their original ids.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// splitmix64 finalizer (the oracle's own copy; pinned by test vectors in
// tests/test_oracle_pins.py).
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

typedef std::vector<uint32_t> Set;  // sorted ascending ids (L) or ordered list (P, Q, R)

struct Acc {
  uint64_t count = 0, hash = 0, tasks = 0, pruned = 0, bad = 0;
};

struct Graph {
  int cand_side = 1;                 // which input side is the candidate side U (P, Q, R ⊆ U)
  std::vector<Set> adjU;             // u ∈ U → sorted N(u) ⊆ V
  std::vector<Set> adjV;             // v ∈ V → sorted N(v) ⊆ U
  std::vector<uint32_t> rank;        // r(u): position of u in ascending (deg, original id)
  int order_mode = 0;                // 0 = ascending (|N(v)∩L|, r(v)); 1 = input order; 2 = descending
  bool check = false;                // verify A = N(B), B = N(A) for every emission
  // optional listing (single-threaded use only)
  std::vector<uint32_t>* listing = nullptr;
};

// |a ∩ b| for two sorted id lists.  Plain merge; binary search of the shorter
// list in the longer one when sizes are very unbalanced (same value).
uint64_t count_common(const Set& a, const Set& b) {
  const Set& s = a.size() <= b.size() ? a : b;
  const Set& l = a.size() <= b.size() ? b : a;
  uint64_t c = 0;
  if (s.size() * 16 < l.size()) {
    for (uint32_t v : s) c += std::binary_search(l.begin(), l.end(), v) ? 1 : 0;
    return c;
  }
  size_t i = 0, j = 0;
  while (i < s.size() && j < l.size()) {
    if (s[i] < l[j]) ++i;
    else if (s[i] > l[j]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

Set intersect(const Set& a, const Set& b) {
  Set out;
  std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
  return out;
}

// Result hash of one biclique (L' ⊆ V, R' ⊆ U), in the input orientation:
// A = side-1 set, B = side-2 set (original ids).
//   sA = Σ mix64(2a), sB = Σ mix64(2b+1),
//   H  = mix64(sA ^ rotl64(sB,32) ^ (|A| << 32) ^ |B|).
uint64_t biclique_hash(const Graph& g, const Set& Lp, const Set& Rp) {
  const Set& A = g.cand_side == 1 ? Rp : Lp;
  const Set& B = g.cand_side == 1 ? Lp : Rp;
  uint64_t sA = 0, sB = 0;
  for (uint32_t a : A) sA += mix64(2ULL * a);
  for (uint32_t b : B) sB += mix64(2ULL * b + 1);
  return mix64(sA ^ rotl64(sB, 32) ^ ((uint64_t)A.size() << 32) ^ (uint64_t)B.size());
}

// Debug check of one emission: R' = N(L') and L' = N(R').
bool closed(const Graph& g, const Set& Lp, const Set& Rp) {
  Set R = Rp;
  std::sort(R.begin(), R.end());
  if (std::adjacent_find(R.begin(), R.end()) != R.end()) return false;
  Set nL = g.adjV[Lp[0]];
  for (size_t k = 1; k < Lp.size(); ++k) nL = intersect(nL, g.adjV[Lp[k]]);
  if (nL != R) return false;
  Set nR = g.adjU[R[0]];
  for (size_t k = 1; k < R.size(); ++k) nR = intersect(nR, g.adjU[R[k]]);
  return nR == Lp;
}

void emit(const Graph& g, const Set& Lp, const Set& Rp, Acc& acc) {
  acc.count += 1;
  acc.hash += biclique_hash(g, Lp, Rp);
  if (g.check && !closed(g, Lp, Rp)) acc.bad += 1;
  if (g.listing) {
    const Set& A = g.cand_side == 1 ? Rp : Lp;
    const Set& B = g.cand_side == 1 ? Lp : Rp;
    Set a = A, b = B;
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    g.listing->push_back((uint32_t)a.size());
    g.listing->push_back((uint32_t)b.size());
    g.listing->insert(g.listing->end(), a.begin(), a.end());
    g.listing->insert(g.listing->end(), b.begin(), b.end());
  }
}

void mbea(const Graph& g, const Set& L, const Set& R, Set P, Set Q, Acc& acc);

// One iteration of the while loop of Algorithm 1 for the popped candidate x,
// with P = the candidates still after x and Q = the current Q.
// L == nullptr means L = V (the root), where L ∩ N(x) = N(x).
void iteration(const Graph& g, const Set* L, const Set& R, uint32_t x, const Set& P, const Set& Q,
               Acc& acc) {
  // Step 1: R' = R ∪ {x}
  Set Rp = R;
  Rp.push_back(x);
  // Step 2: L' = {v ∈ L : (x, v) ∈ E}
  Set Lp = L ? intersect(*L, g.adjU[x]) : g.adjU[x];
  if (Lp.empty()) return;  // reading Z1
  acc.tasks += 1;
  // Step 3: maximality check over Q
  Set Qp;
  for (uint32_t v : Q) {
    uint64_t c = count_common(g.adjU[v], Lp);
    if (c == Lp.size()) { acc.pruned += 1; return; }  // not maximal
    if (c > 0) Qp.push_back(v);
  }
  // Step 4: maximal expansion over P
  std::vector<std::pair<uint64_t, uint32_t>> Pk;  // (key, v)
  for (uint32_t v : P) {
    uint64_t c = count_common(g.adjU[v], Lp);
    if (c == Lp.size()) Rp.push_back(v);
    else if (c > 0) Pk.push_back({((g.order_mode == 2 ? (0xffffffffULL - c) : c) << 32) | g.rank[v], v});
  }
  emit(g, Lp, Rp, acc);
  if (!Pk.empty()) {
    // next-level order (reading Z6): ascending (|N(v) ∩ L'|, r(v)); input order keeps P's order;
    // descending (-|N(v) ∩ L'|, r(v))
    if (g.order_mode != 1) std::sort(Pk.begin(), Pk.end());
    Set Pp;
    Pp.reserve(Pk.size());
    for (auto& kv : Pk) Pp.push_back(kv.second);
    mbea(g, Lp, Rp, Pp, Qp, acc);
  }
}

// MBEA(L, R, P, Q), Algorithm 1.
void mbea(const Graph& g, const Set& L, const Set& R, Set P, Set Q, Acc& acc) {
  size_t head = 0;
  while (head < P.size()) {       // while |P| > 0
    uint32_t x = P[head++];       // x = P.pop()
    Set rest(P.begin() + head, P.end());
    iteration(g, &L, R, x, rest, Q, acc);
    Q.push_back(x);               // Q = Q ∪ {x}
  }
}

// Root iteration i of the top-level loop: x = root[i], Q = root[0..i-1],
// P = root[i+1..], L = V, R = ∅ — restricted to N(N(x)) (exact, see header).
void root_iteration(const Graph& g, const std::vector<uint32_t>& root, const std::vector<uint32_t>& pos,
                    size_t i, std::vector<uint32_t>& mark, Acc& acc) {
  uint32_t x = root[i];
  // 2-hop H = ∪_{u ∈ N(x)} N(u), listed in root order (the order Q and P hold).
  std::vector<uint32_t> H;
  for (uint32_t u : g.adjU[x])
    for (uint32_t v : g.adjV[u])
      if (!mark[v] && v != x) { mark[v] = 1; H.push_back(v); }
  for (uint32_t v : H) mark[v] = 0;
  std::sort(H.begin(), H.end(), [&](uint32_t a, uint32_t b) { return pos[a] < pos[b]; });
  Set Q, P;
  for (uint32_t v : H) {
    if (pos[v] == UINT32_MAX) continue;  // degree 0 cannot be in H; defensive
    (pos[v] < i ? Q : P).push_back(v);
  }
  iteration(g, nullptr, Set(), x, P, Q, acc);
}

int build(Graph& g, uint32_t n1, uint32_t n2, const uint64_t* row_ptr, const uint32_t* col_idx,
          int candidate_side) {
  for (uint32_t i = 0; i < n1; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return -1;
  uint64_t nnz = n1 ? row_ptr[n1] : 0;
  for (uint64_t e = 0; e < nnz; ++e)
    if (col_idx[e] >= n2) return -5;
  int side = candidate_side;
  if (side == 0) side = (n2 < n1) ? 2 : 1;  // smaller side; ties keep side 1 (reading Z4)
  g.cand_side = side;
  uint32_t nU = side == 1 ? n1 : n2, nV = side == 1 ? n2 : n1;
  g.adjU.assign(nU, Set());
  g.adjV.assign(nV, Set());
  for (uint32_t i = 0; i < n1; ++i)
    for (uint64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      uint32_t j = col_idx[e];
      if (side == 1) { g.adjU[i].push_back(j); g.adjV[j].push_back(i); }
      else { g.adjU[j].push_back(i); g.adjV[i].push_back(j); }
    }
  for (auto& s : g.adjU) { std::sort(s.begin(), s.end()); s.erase(std::unique(s.begin(), s.end()), s.end()); }
  for (auto& s : g.adjV) { std::sort(s.begin(), s.end()); s.erase(std::unique(s.begin(), s.end()), s.end()); }
  std::vector<uint32_t> byrank(nU);
  for (uint32_t u = 0; u < nU; ++u) byrank[u] = u;
  std::sort(byrank.begin(), byrank.end(), [&](uint32_t a, uint32_t b) {
    if (g.adjU[a].size() != g.adjU[b].size()) return g.adjU[a].size() < g.adjU[b].size();
    return a < b;
  });
  g.rank.assign(nU, 0);
  for (uint32_t k = 0; k < nU; ++k) g.rank[byrank[k]] = k;
  return 0;
}

// Root P: degree ≥ 1 vertices, ascending (deg, id), input (id) or descending (-deg, id) order.
// r(v) (g.rank) is the position of v in that order, the tie-break of every later level.
std::vector<uint32_t> root_order(Graph& g) {
  const uint32_t nU = (uint32_t)g.adjU.size();
  std::vector<uint32_t> all(nU);
  for (uint32_t u = 0; u < nU; ++u) all[u] = u;
  if (g.order_mode == 2)
    std::sort(all.begin(), all.end(), [&](uint32_t a, uint32_t b) {
      if (g.adjU[a].size() != g.adjU[b].size()) return g.adjU[a].size() > g.adjU[b].size();
      return a < b;
    });
  else if (g.order_mode == 0)
    std::sort(all.begin(), all.end(), [&](uint32_t a, uint32_t b) { return g.rank[a] < g.rank[b]; });
  for (uint32_t k = 0; k < nU; ++k) g.rank[all[k]] = k;
  std::vector<uint32_t> root;
  for (uint32_t u : all)
    if (!g.adjU[u].empty()) root.push_back(u);
  return root;
}

}  // namespace

extern "C" {

// Full enumeration.  out[0..4] = count, hash, tasks, pruned, bad (closure-check failures).
// candidate_side: 0 auto (smaller side), 1 rows, 2 cols.  order_mode: 0 ascending, 1 input.
// threads: 0 = hardware_concurrency.  Returns 0, or -1 (row_ptr non-monotone) / -5 (col id ≥ n2).
int oracle_mbea(uint32_t n1, uint32_t n2, const uint64_t* row_ptr, const uint32_t* col_idx,
                int candidate_side, int order_mode, int threads, int check, uint64_t* out) {
  Graph g;
  int rc = build(g, n1, n2, row_ptr, col_idx, candidate_side);
  if (rc) return rc;
  g.order_mode = order_mode;
  g.check = check != 0;
  std::vector<uint32_t> root = root_order(g);
  std::vector<uint32_t> pos(g.adjU.size(), UINT32_MAX);
  for (size_t k = 0; k < root.size(); ++k) pos[root[k]] = (uint32_t)k;
  unsigned nt = threads > 0 ? (unsigned)threads : std::max(1u, std::thread::hardware_concurrency());
  std::atomic<size_t> next(0);
  std::vector<Acc> accs(nt);
  auto worker = [&](unsigned t) {
    std::vector<uint32_t> mark(g.adjU.size(), 0);
    for (;;) {
      size_t i = next.fetch_add(1);
      if (i >= root.size()) break;
      root_iteration(g, root, pos, i, mark, accs[t]);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  Acc tot;
  for (auto& a : accs) {
    tot.count += a.count; tot.hash += a.hash; tot.tasks += a.tasks; tot.pruned += a.pruned; tot.bad += a.bad;
  }
  out[0] = tot.count; out[1] = tot.hash; out[2] = tot.tasks; out[3] = tot.pruned; out[4] = tot.bad;
  out[5] = nt;
  return 0;
}

// Per-root results for selected candidate-side vertices (original ids):
// per_root[4*k + {0,1,2,3}] = count, hash, tasks, pruned of the level-1
// subtree of roots[k] (all zeros for a degree-0 vertex).  Must use the same
// candidate_side/order as the run being compared.
int oracle_mbea_roots(uint32_t n1, uint32_t n2, const uint64_t* row_ptr, const uint32_t* col_idx,
                      int candidate_side, int order_mode, int threads, const uint32_t* roots,
                      uint64_t n_roots, uint64_t* per_root) {
  Graph g;
  int rc = build(g, n1, n2, row_ptr, col_idx, candidate_side);
  if (rc) return rc;
  g.order_mode = order_mode;
  for (uint64_t k = 0; k < n_roots; ++k)
    if (roots[k] >= g.adjU.size()) return -5;
  std::vector<uint32_t> root = root_order(g);
  std::vector<uint32_t> pos(g.adjU.size(), UINT32_MAX);
  for (size_t k = 0; k < root.size(); ++k) pos[root[k]] = (uint32_t)k;
  unsigned nt = threads > 0 ? (unsigned)threads : std::max(1u, std::thread::hardware_concurrency());
  std::atomic<uint64_t> next(0);
  auto worker = [&]() {
    std::vector<uint32_t> mark(g.adjU.size(), 0);
    for (;;) {
      uint64_t k = next.fetch_add(1);
      if (k >= n_roots) break;
      Acc a;
      uint32_t x = roots[k];
      if (pos[x] != UINT32_MAX) root_iteration(g, root, pos, pos[x], mark, a);
      per_root[4 * k + 0] = a.count; per_root[4 * k + 1] = a.hash;
      per_root[4 * k + 2] = a.tasks; per_root[4 * k + 3] = a.pruned;
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return 0;
}

// Listing (single thread, small graphs): writes records [|A|, |B|, A ids..., B ids...]
// (original ids, each side ascending) into buf (cap words).  Returns the number
// of words needed (may exceed cap: then buf holds a prefix), or a negative error.
int64_t oracle_mbea_list(uint32_t n1, uint32_t n2, const uint64_t* row_ptr, const uint32_t* col_idx,
                         int candidate_side, int order_mode, uint32_t* buf, uint64_t cap) {
  Graph g;
  int rc = build(g, n1, n2, row_ptr, col_idx, candidate_side);
  if (rc) return rc;
  g.order_mode = order_mode;
  std::vector<uint32_t> listing;
  g.listing = &listing;
  std::vector<uint32_t> root = root_order(g);
  Acc acc;
  // Plain sequential top-level MBEA(V, ∅, root P, ∅) — no 2-hop shortcut here.
  Set L(g.adjV.size());
  for (uint32_t v = 0; v < L.size(); ++v) L[v] = v;
  mbea(g, L, Set(), root, Set(), acc);
  uint64_t n = std::min<uint64_t>(cap, listing.size());
  if (n) std::memcpy(buf, listing.data(), n * sizeof(uint32_t));
  return (int64_t)listing.size();
}

// Sequential full MBEA without the root 2-hop shortcut (small graphs): the
// literal top-level call MBEA(V, ∅, P, ∅).  out as oracle_mbea.
int oracle_mbea_plain(uint32_t n1, uint32_t n2, const uint64_t* row_ptr, const uint32_t* col_idx,
                      int candidate_side, int order_mode, uint64_t* out) {
  Graph g;
  int rc = build(g, n1, n2, row_ptr, col_idx, candidate_side);
  if (rc) return rc;
  g.order_mode = order_mode;
  g.check = true;
  std::vector<uint32_t> root = root_order(g);
  Acc acc;
  Set L(g.adjV.size());
  for (uint32_t v = 0; v < L.size(); ++v) L[v] = v;
  mbea(g, L, Set(), root, Set(), acc);
  out[0] = acc.count; out[1] = acc.hash; out[2] = acc.tasks; out[3] = acc.pruned; out[4] = acc.bad;
  out[5] = 1;
  return 0;
}

uint64_t oracle_mix64(uint64_t z) { return mix64(z); }

}  // extern "C"
