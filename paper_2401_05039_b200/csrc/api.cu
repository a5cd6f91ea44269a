// api.cu — C-ABI of libmbe (include/mbe.h): ingest, device memory, launch.
//
// Ingest (one-time, outside the timed search): both CSR
// directions sorted and deduplicated (reading Z8), the candidate side U
// relabelled by ascending (degree, original id) so that rank order is the
// iMBE root order and "Q-role at the root" is "rank < x", the
// per-vertex hash terms hv, and the execution order of the level-1 subtrees
// (a scheduling heuristic, result-invariant: descending estimated P-role
// 2-hop size).  The search itself runs in search.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mbe.h"
#include "bits.cuh"
#include "mbe_internal.h"

namespace {

thread_local std::string g_detail;

int fail(int code, const std::string& msg) {
  g_detail = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess) return fail(MBE_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

thread_local uint64_t* g_upload_counter = nullptr;
thread_local unsigned g_ingest_threads = 0;  // mbe_load_csr flags bits 0-7 (0 = auto)

// Host ingest threads: the mbe_load_csr flags request, else min(hardware threads, 16); 1 for small graphs.
unsigned ingest_threads(uint64_t work) {
  if (g_ingest_threads) return g_ingest_threads;
  if (work < (1u << 16)) return 1;
  const unsigned h = std::thread::hardware_concurrency();
  return std::min(16u, std::max(1u, h));
}

// fn(t, begin, end) over T contiguous ranges of [0, n); range t = [n t / T, n (t + 1) / T).
template <class F>
void parallel_ranges(uint64_t n, unsigned T, F&& fn) {
  if (T <= 1 || n < T) {
    fn(0u, (uint64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T - 1);
  for (unsigned t = 1; t < T; ++t) th.emplace_back([&fn, n, T, t] { fn(t, n * t / T, n * (t + 1) / T); });
  fn(0u, (uint64_t)0, n / T);
  for (auto& x : th) x.join();
}

// fn(t, begin, end) over T vertex ranges of [0, n) holding about equal numbers of edges (off = CSR offsets,
// n + 1 entries): power-law degrees put most edges on few vertices, so equal vertex counts load-imbalance.
template <class Off, class F>
void parallel_edges(const Off* off, uint64_t n, unsigned T, F&& fn) {
  if (T <= 1 || n < T) {
    fn(0u, (uint64_t)0, n);
    return;
  }
  std::vector<uint64_t> cut(T + 1, n);
  cut[0] = 0;
  const uint64_t E = off[n] - off[0];
  for (unsigned t = 1; t < T; ++t)
    cut[t] = (uint64_t)(std::lower_bound(off, off + n + 1, (Off)(off[0] + E * t / T)) - off);
  for (unsigned t = 1; t <= T; ++t) cut[t] = std::max(cut[t], cut[t - 1]);
  std::vector<std::thread> th;
  th.reserve(T - 1);
  for (unsigned t = 1; t < T; ++t) th.emplace_back([&fn, &cut, t] { fn(t, cut[t], cut[t + 1]); });
  fn(0u, cut[0], cut[1]);
  for (auto& x : th) x.join();
}

// Pinned staging buffer for the one H2D copy of a side's packed arrays (kept across loads).
std::mutex g_stage_mu;
void* g_stage = nullptr;
size_t g_stage_bytes = 0;

// Device blocks of freed graphs, kept for the next mbe_load_csr (a caching allocator: cudaFree
// synchronises the device and was measured at 2-460 ms per mbe_free with the search workspaces
// resident).  Returned to the driver by mbe_release_workspaces.
struct CachedBlock {
  int device;
  void* p;
  size_t bytes;
};
std::mutex g_graph_cache_mu;
std::vector<CachedBlock> g_graph_cache;

int graph_alloc(DevBuf& b, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_graph_cache_mu);
    size_t best = SIZE_MAX;
    for (size_t k = 0; k < g_graph_cache.size(); ++k) {
      const CachedBlock& c = g_graph_cache[k];
      if (c.device == dev && c.bytes >= bytes && c.bytes <= 2 * bytes + (1u << 20) &&
          (best == SIZE_MAX || c.bytes < g_graph_cache[best].bytes))
        best = k;
    }
    if (best != SIZE_MAX) {
      b.p = g_graph_cache[best].p;
      b.bytes = g_graph_cache[best].bytes;
      g_graph_cache.erase(g_graph_cache.begin() + best);
      return MBE_OK;
    }
  }
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return fail(MBE_ENOMEM, "cudaMalloc graph");
  }
  b.bytes = bytes;
  return MBE_OK;
}

void graph_release(DevBuf& b) {
  if (b.p) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_graph_cache_mu);
    g_graph_cache.push_back({dev, b.p, b.bytes});
  }
  b.p = nullptr;
  b.bytes = 0;
}


struct Side {
  bool built = false;
  bool twin_ready = false;      // root twin flags computed (graph-only, once per side)
  uint32_t auto_T = 0;          // cached auto bit-row threshold
  uint32_t nU = 0, nV = 0, n_roots = 0, maxdegU = 0;
  uint64_t cand = 0;            // max |N(N(x))| over candidates x: bounds every task's candidate buffers
  std::vector<uint32_t> origU;  // host copy: rank -> original id
  std::vector<uint32_t> rankU;  // host copy: original id -> rank
  DevBuf all;                   // one device allocation holding every array below
  DevBuf offU, adjU, offV, adjV, hvU, hvV, origUd, root_order, twin;  // views into `all` (not owned)
  void release() {
    graph_release(all);
    for (DevBuf* b : {&offU, &adjU, &offV, &adjV, &hvU, &hvV, &origUd, &root_order, &twin}) *b = DevBuf();
    built = false;
  }
};

// Host->device copies of ingest run on a per-device NON-BLOCKING stream: a load on one host thread then
// never waits for a search running on another thread's stream (the legacy default stream would).
cudaStream_t copy_stream() {
  static std::mutex mu;
  static cudaStream_t s[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!s[dev] && cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    s[dev] = nullptr;
  }
  return s[dev];
}

int copy_h2d(void* dst, const void* src, size_t bytes) {
  cudaStream_t cs = copy_stream();
  if (!cs) {
    CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return MBE_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs));
  CUDA_TRY(cudaStreamSynchronize(cs));
  return MBE_OK;
}

// Packs host arrays into one device allocation (one cudaMalloc, one cudaFree per side).
struct Packer {
  struct Item { DevBuf* dst; const void* src; size_t bytes; size_t off; };
  std::vector<Item> items;
  size_t total = 0;
  void add(DevBuf& dst, const void* src, size_t bytes) {
    items.push_back({&dst, src, bytes, total});
    total += (std::max<size_t>(bytes, 16) + 255) & ~size_t(255);
  }
  int commit(DevBuf& all, uint64_t* counter) {
    if (int rc = graph_alloc(all, std::max<size_t>(total, 256))) return rc;
    for (const Item& it : items) {
      it.dst->p = static_cast<uint8_t*>(all.p) + it.off;
      it.dst->bytes = it.bytes;
      if (counter && it.src) *counter += it.bytes;
    }
    std::lock_guard<std::mutex> lk(g_stage_mu);
    if (g_stage_bytes < total) {
      if (g_stage) cudaFreeHost(g_stage);
      g_stage = nullptr;
      g_stage_bytes = 0;
      const size_t want = total + total / 4;
      if (cudaHostAlloc(&g_stage, want, cudaHostAllocDefault) == cudaSuccess) {
        g_stage_bytes = want;
      } else {
        cudaGetLastError();
        g_stage = nullptr;
      }
    }
    if (!g_stage) {  // no pinned memory: pageable copies straight from the arrays
      for (const Item& it : items)
        if (it.src && it.bytes)
          if (int rc = copy_h2d(it.dst->p, it.src, it.bytes)) return rc;
      return MBE_OK;
    }
    uint8_t* stage = static_cast<uint8_t*>(g_stage);
    // parallel gather into the staging buffer: 1 MiB chunks of every item, dealt over the threads
    std::vector<std::pair<size_t, size_t>> chunks;  // (item, byte offset in the item)
    for (size_t k = 0; k < items.size(); ++k)
      if (items[k].src)
        for (size_t o = 0; o < items[k].bytes; o += (1u << 20)) chunks.push_back({k, o});
    parallel_ranges(chunks.size(), ingest_threads(total / 4), [&](unsigned, uint64_t a, uint64_t b) {
      for (uint64_t c = a; c < b; ++c) {
        const Item& it = items[chunks[c].first];
        const size_t o = chunks[c].second, n = std::min<size_t>(1u << 20, it.bytes - o);
        std::memcpy(stage + it.off + o, static_cast<const uint8_t*>(it.src) + o, n);
      }
    });
    return copy_h2d(all.p, stage, total);
  }
};

// Search workspace (per-warp scratch + frame arenas + descriptors).  Pooled
// process-wide per device and checked out exclusively by one mbe_enumerate
// call at a time, so load -> enumerate -> free cycles do not re-allocate GBs.
struct Workspace {
  int device = 0;
  bool busy = false, dirty = true;
  uint32_t n_warps = 0, wmax = 0;
  uint64_t cap_nU = 0, cap_cand = 0, cap_lbuf = 0, arena_bytes = 0, stride = 0;
  uint64_t o_slot = 0, o_crow = 0, o_touched = 0, o_lbuf = 0, o_rbuf = 0, o_skey = 0, o_sval = 0, o_pbuf = 0, o_qbuf = 0,
           o_arena = 0;
  DevBuf ws, desc, tops, stamps, hint, per_root, gl;
  void release() {
    for (DevBuf* b : {&ws, &desc, &tops, &stamps, &hint, &per_root, &gl}) b->release();
  }
};

std::mutex g_pool_mu;
std::vector<Workspace*> g_pool;

}  // namespace

struct mbe_graph {
  int device = 0;
  uint32_t n1 = 0, n2 = 0;
  uint64_t nE = 0;
  // deduplicated host CSR in both directions (original ids)
  std::vector<uint32_t> off1, adj1, off2, adj2;
  Side side[2][3];  // [candidate side - 1][candidate order]
  uint64_t h2d_bytes = 0;  // bytes uploaded by ingest (all built sides)
  SearchParams sp;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int sm_count = 0;
  int occ[2][5] = {{0}};         // cached occupancy: [instr][threads/32 - 1] resident CTAs per SM
  DevBuf claim_tab;             // shared-counter claim log of the current call ([n_roots + 1] u64)
  ~mbe_graph();
};

// Timing events and SM counts are process-wide per device: creating or destroying an event (or querying an
// attribute) can wait for a search kernel running on another thread, which would serialise a loader thread
// with the search it is meant to overlap.  Events come from a pool (filled lazily by mbe_enumerate).
std::mutex g_ev_mu;
std::vector<std::pair<int, cudaEvent_t>> g_ev_pool;
cudaEvent_t ev_get(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_ev_mu);
    for (size_t k = 0; k < g_ev_pool.size(); ++k)
      if (g_ev_pool[k].first == dev) {
        cudaEvent_t e = g_ev_pool[k].second;
        g_ev_pool.erase(g_ev_pool.begin() + k);
        return e;
      }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}
void ev_put(int dev, cudaEvent_t e) {
  if (!e) return;
  std::lock_guard<std::mutex> lk(g_ev_mu);
  g_ev_pool.push_back({dev, e});
}
int sm_count_of(int dev) {
  static std::mutex mu;
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 0;
  std::lock_guard<std::mutex> lk(mu);
  if (!cache[dev] && cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    cache[dev] = 0;
  }
  return cache[dev];
}

mbe_graph::~mbe_graph() {
  claim_tab.release();
  for (auto& so : side)
    for (auto& s : so) s.release();
  ev_put(device, ev0);
  ev_put(device, ev1);
}

namespace {

// Build the device graph for candidate side s (1 = rows, 2 = cols).
int build_side(mbe_graph* g, int s, uint32_t order = 0) {
  Side& S = g->side[s - 1][order];
  if (S.built) return MBE_OK;
  g_upload_counter = &g->h2d_bytes;
  const bool dbg = std::getenv("MBE_DEBUG_TIMING") != nullptr;
  auto T = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "    side %-26s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - T).count());
    T = n;
  };
  const std::vector<uint32_t>& offC = s == 1 ? g->off1 : g->off2;  // candidate side CSR
  const std::vector<uint32_t>& adjC = s == 1 ? g->adj1 : g->adj2;
  const uint32_t nU = s == 1 ? g->n1 : g->n2, nV = s == 1 ? g->n2 : g->n1;
  S.nU = nU;
  S.nV = nV;
  // rank = position in the root order: ascending (degree, original id) by a counting sort over degrees
  // (stable in id); descending (-degree, id) by the same sort over maxdeg - degree; input = original id
  uint32_t maxdeg = 0;
  for (uint32_t u = 0; u < nU; ++u) maxdeg = std::max(maxdeg, offC[u + 1] - offC[u]);
  auto dkey = [&](uint32_t u) {
    const uint32_t d = offC[u + 1] - offC[u];
    return order == 2 ? maxdeg - d : (order == 1 ? 0u : d);
  };
  std::vector<uint32_t> bucket(maxdeg + 2, 0);
  for (uint32_t u = 0; u < nU; ++u) bucket[dkey(u) + 1]++;
  for (uint32_t d = 1; d < bucket.size(); ++d) bucket[d] += bucket[d - 1];
  S.origU.assign(nU, 0);
  S.rankU.assign(nU, 0);
  for (uint32_t u = 0; u < nU; ++u) {
    uint32_t r = bucket[dkey(u)]++;
    S.origU[r] = u;
    S.rankU[u] = r;
  }
  S.maxdegU = maxdeg;
  lap("relabel");
  // adjU[rank] = sorted V ids; adjV[v] = sorted ranks (the other direction's CSR mapped through
  // rankU, each row re-sorted); all passes are parallel over vertex ranges
  const unsigned nth = ingest_threads(g->nE);
  if (dbg) std::fprintf(stderr, "    side ingest threads %u\n", nth);
  const std::vector<uint32_t>& offO = s == 1 ? g->off2 : g->off1;  // other side's CSR (candidate ids)
  const std::vector<uint32_t>& adjO = s == 1 ? g->adj2 : g->adj1;
  std::vector<uint32_t> offU(nU + 1, 0), adjU(g->nE), offV(offO.begin(), offO.end()), adjV(g->nE);
  for (uint32_t r = 0; r < nU; ++r) {
    const uint32_t u = S.origU[r];
    offU[r + 1] = offU[r] + (offC[u + 1] - offC[u]);
  }
  parallel_edges(offU.data(), nU, nth, [&](unsigned, uint64_t a, uint64_t b) {
    for (uint64_t r = a; r < b; ++r) {
      const uint32_t u = S.origU[r];
      std::copy(adjC.begin() + offC[u], adjC.begin() + offC[u + 1], adjU.begin() + offU[r]);
    }
  });
  lap("adjacency: offU + adjU");
  parallel_edges(offV.data(), nV, nth, [&](unsigned, uint64_t a, uint64_t b) {
    for (uint64_t v = a; v < b; ++v) {
      for (uint32_t e = offV[v]; e < offV[v + 1]; ++e) adjV[e] = S.rankU[adjO[e]];
      std::sort(adjV.begin() + offV[v], adjV.begin() + offV[v + 1]);
    }
  });
  // execution-order cost of each level-1 subtree (descending P-role 2-hop estimate):
  //   cost(x) = Σ_{u ∈ N(x)} |{w ∈ N(u) : w > x}| = Σ_{u ∈ N(x)} deg(u) - k - 1, k = position of x in adjV[u]
  lap("adjacency: adjV");
  std::vector<uint64_t> rcost(nU, 0), vis(nU, 0);
  parallel_edges(offU.data(), nU, nth, [&](unsigned, uint64_t a, uint64_t b) {
    for (uint64_t r = a; r < b; ++r) {
      uint64_t c = 0, v = 0;
      for (uint32_t e = offU[r]; e < offU[r + 1]; ++e) {
        const uint32_t u = adjU[e];
        const uint32_t k = (uint32_t)(std::lower_bound(adjV.begin() + offV[u], adjV.begin() + offV[u + 1], (uint32_t)r) -
                                      adjV.begin());
        c += offV[u + 1] - k - 1;
        v += offV[u + 1] - offV[u];
      }
      rcost[r] = c;
      vis[r] = v;
    }
  });
  // Candidate-buffer bound: the largest 2-hop set |N(N(x))| (x included).  Every vertex a task in x's
  // level-1 subtree touches, classifies or keeps as a P'/Q' row lies in N(N(x)) (L' ⊆ N(x) below the
  // root), so it bounds the per-warp touched list, R', sort keys and P'/Q' rows.  |N(N(x))| <= vis(x) =
  // Σ_{u ∈ N(x)} deg(u), so exact sizes are computed only for candidates, by descending vis, while vis
  // can still beat the best found (a few dozen on power-law graphs).
  {
    auto two_hop = [&](uint32_t r, std::vector<uint32_t>& stamp) {
      uint64_t two = 0;
      for (uint32_t e = offU[r]; e < offU[r + 1]; ++e)
        for (uint32_t f = offV[adjU[e]]; f < offV[adjU[e] + 1]; ++f)
          if (stamp[adjV[f]] != r) {
            stamp[adjV[f]] = r;
            ++two;
          }
      return two;
    };
    uint32_t top = 0;
    for (uint32_t r = 1; r < nU; ++r)
      if (vis[r] > vis[top]) top = r;
    std::vector<uint32_t> stamp0(nU, 0xffffffffu);
    std::atomic<uint64_t> best(nU ? two_hop(top, stamp0) : 0);
    std::vector<std::pair<uint64_t, uint32_t>> cand;  // candidates that could still beat it, by descending vis
    for (uint32_t r = 0; r < nU; ++r)
      if (r != top && vis[r] > best.load()) cand.emplace_back(vis[r], r);
    std::sort(cand.begin(), cand.end(), std::greater<>());
    std::atomic<size_t> next(0);
    auto worker = [&](std::vector<uint32_t>& stamp) {
      for (size_t k; (k = next.fetch_add(1)) < cand.size();) {
        if (cand[k].first <= best.load()) break;  // sorted: no later candidate can beat the best
        const uint64_t two = two_hop(cand[k].second, stamp);
        for (uint64_t b = best.load(); two > b && !best.compare_exchange_weak(b, two);) {
        }
      }
    };
    const unsigned T = std::max(1u, std::min<unsigned>(nth, (unsigned)cand.size()));
    std::vector<std::thread> th;
    std::vector<std::vector<uint32_t>> stamps(T > 1 ? T - 1 : 0, std::vector<uint32_t>(nU, 0xffffffffu));
    for (unsigned t = 1; t < T; ++t) th.emplace_back(worker, std::ref(stamps[t - 1]));
    worker(stamp0);
    for (auto& x : th) x.join();
    S.cand = best.load();
  }
  lap("adjacency");
  // hash terms: side bit 0 for side 1 (rows), 1 for side 2 (cols)
  std::vector<uint64_t> hvU(nU), hvV(nV);
  const uint64_t bu = s == 1 ? 0 : 1, bv = 1 - bu;
  for (uint32_t r = 0; r < nU; ++r) hvU[r] = mbe_mix64(2ull * S.origU[r] + bu);
  for (uint32_t v = 0; v < nV; ++v) hvV[v] = mbe_mix64(2ull * v + bv);
  lap("hash terms");
  // execution order: descending cost, ties by rank (one u64 key per root)
  std::vector<uint64_t> key;
  key.reserve(nU);
  for (uint32_t r = 0; r < nU; ++r) {
    if (offU[r + 1] == offU[r]) continue;
    const uint64_t c = std::min<uint64_t>(rcost[r], 0xffffffffull);
    key.push_back(((0xffffffffull - c) << 32) | r);
  }
  {  // LSD radix sort, 16-bit digits (4 stable passes; std::sort took ~5 ms for 10^5 keys)
    std::vector<uint64_t> tmp(key.size());
    std::vector<uint32_t> cnt(1u << 16);
    for (int sh = 0; sh < 64; sh += 16) {
      std::fill(cnt.begin(), cnt.end(), 0u);
      for (uint64_t k : key) cnt[(k >> sh) & 0xffffu]++;
      uint32_t run = 0;
      for (uint32_t& c : cnt) {
        const uint32_t n = c;
        c = run;
        run += n;
      }
      for (uint64_t k : key) tmp[cnt[(k >> sh) & 0xffffu]++] = k;
      key.swap(tmp);
    }
  }
  lap("root cost + sort");
  std::vector<uint32_t> exec(key.size());  // execution order of the level-1 subtrees
  for (size_t k = 0; k < key.size(); ++k) exec[k] = (uint32_t)key[k];
  S.n_roots = (uint32_t)exec.size();
  Packer pk;
  pk.add(S.offU, offU.data(), offU.size() * 4);
  pk.add(S.adjU, adjU.data(), adjU.size() * 4);
  pk.add(S.offV, offV.data(), offV.size() * 4);
  pk.add(S.adjV, adjV.data(), adjV.size() * 4);
  pk.add(S.hvU, hvU.data(), hvU.size() * 8);
  pk.add(S.hvV, hvV.data(), hvV.size() * 8);
  pk.add(S.origUd, S.origU.data(), S.origU.size() * 4);
  pk.add(S.root_order, exec.data(), exec.size() * 4);
  pk.add(S.twin, nullptr, nU);  // written by the twin pre-pass
  int rc = pk.commit(S.all, g_upload_counter);
  if (rc) {
    S.release();
    return rc;
  }
  lap("pack + upload");
  S.built = true;
  return MBE_OK;
}

uint64_t align256(uint64_t x) { return (x + 255) & ~255ull; }

// Per-warp workspace layout (bytes from the warp's base).  The hot, small-index parts of every scratch
// buffer sit next to each other (arena first, then the candidate-indexed buffers), and the two
// vertex-indexed slot table (random access by vertex id) comes last.  `cand` bounds the rows of any one
// task's candidate buffers (the reverse scan's compact bit rows, touched, R', sort keys, P'/Q' rows).
struct WsLayout {
  uint64_t slot, crow, touched, lbuf, rbuf, skey, sval, pbuf, qbuf, arena, stride;
};
WsLayout ws_layout(uint64_t nU, uint64_t cand, uint64_t maxdeg, uint64_t arena_bytes, uint32_t wmax) {
  nU = std::max<uint64_t>(nU, 1);
  cand = std::max<uint64_t>(std::min(cand, nU), 1);
  const uint64_t lb = std::max<uint64_t>(maxdeg, 32 * MBE_WMAX);
  WsLayout L;
  uint64_t o = 0;
  L.arena = o; o = align256(o + arena_bytes);
  L.crow = o; o = align256(o + (wmax > 4 ? cand * 4 * MBE_CROW_WORDS : 0));
  L.touched = o; o = align256(o + cand * 4);
  L.lbuf = o; o = align256(o + lb * 4);
  L.rbuf = o; o = align256(o + cand * 4);
  L.skey = o; o = align256(o + cand * 32);  // sort keys + ping-pong copy, or a dedup hash table of <= 4 cand u64
  L.sval = o; o = align256(o + cand * 8);
  L.pbuf = o; o = align256(o + cand * wmax * 4);
  L.qbuf = o; o = align256(o + cand * wmax * 4);
  L.slot = o; o = align256(o + nU * 4 * MBE_SLOT_WORDS);
  L.stride = o;
  return L;
}

uint64_t workspace_stride(uint64_t nU, uint64_t cand, uint64_t maxdeg, uint64_t arena_bytes, uint32_t wmax) {
  return ws_layout(nU, cand, maxdeg, arena_bytes, wmax).stride;
}

// Check out a workspace able to run n_warps warps over nU candidate vertices.
int checkout_workspace(int device, uint32_t n_warps, uint64_t nU, uint64_t cand, uint64_t maxdeg, uint64_t arena_bytes,
                       uint32_t wmax, Workspace** out) {
  nU = std::max<uint64_t>(nU, 1);
  cand = std::max<uint64_t>(std::min(cand, nU), 1);
  const uint64_t lb = std::max<uint64_t>(maxdeg, 32 * MBE_WMAX);
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (Workspace* w : g_pool)
      if (!w->busy && w->device == device && w->n_warps == n_warps && w->cap_nU >= nU && w->cap_cand >= cand &&
          w->cap_lbuf >= lb && w->arena_bytes == arena_bytes && w->wmax >= wmax) {
        w->busy = true;
        *out = w;
        return MBE_OK;
      }
  }
  Workspace* w = new Workspace();
  w->device = device;
  w->n_warps = n_warps;
  w->wmax = wmax;
  w->cap_nU = nU;
  w->cap_cand = cand;
  w->cap_lbuf = lb;
  w->arena_bytes = arena_bytes;
  const WsLayout L = ws_layout(nU, cand, maxdeg, arena_bytes, wmax);
  w->o_slot = L.slot;
  w->o_crow = L.crow;
  w->o_touched = L.touched;
  w->o_lbuf = L.lbuf;
  w->o_rbuf = L.rbuf;
  w->o_skey = L.skey;
  w->o_sval = L.sval;
  w->o_pbuf = L.pbuf;
  w->o_qbuf = L.qbuf;
  w->o_arena = L.arena;
  w->stride = L.stride;
  const uint64_t o = L.stride;
  const uint64_t total = o * n_warps;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (cudaMalloc(&w->ws.p, total) == cudaSuccess) break;
    cudaGetLastError();
    w->ws.p = nullptr;
    if (attempt == 0) {  // free idle pooled workspaces of this device and retry once
      std::lock_guard<std::mutex> lk(g_pool_mu);
      for (auto it = g_pool.begin(); it != g_pool.end();) {
        if (!(*it)->busy && (*it)->device == device) {
          (*it)->release();
          delete *it;
          it = g_pool.erase(it);
        } else {
          ++it;
        }
      }
    }
  }
  if (!w->ws.p) {
    delete w;
    return fail(MBE_ENOMEM, "workspace of " + std::to_string(total >> 20) + " MiB (" + std::to_string(n_warps) +
                                " warps): reduce ctas_per_sm/threads_per_cta/arena_bytes");
  }
  w->ws.bytes = total;
  if (cudaMalloc(&w->desc.p, sizeof(Desc) * MBE_MAXDEPTH * n_warps) != cudaSuccess ||
      cudaMalloc(&w->tops.p, 4ull * n_warps) != cudaSuccess || cudaMalloc(&w->stamps.p, 4ull * n_warps) != cudaSuccess ||
      cudaMalloc(&w->hint.p, 4ull * ((n_warps + 31) / 32)) != cudaSuccess ||
      cudaMalloc(&w->per_root.p, 32ull * nU) != cudaSuccess || cudaMalloc(&w->gl.p, sizeof(Globals)) != cudaSuccess) {
    cudaGetLastError();
    w->release();
    delete w;
    return fail(MBE_ENOMEM, "workspace descriptors");
  }
  w->busy = true;
  w->dirty = true;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(w);
  }
  *out = w;
  return MBE_OK;
}

void checkin_workspace(Workspace* w) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  w->busy = false;
}

// zero the per-vertex slots (required invariant: zero between tasks) and the tag stamps
int clear_tables(Workspace* w, cudaStream_t st) {
  CUDA_TRY(cudaMemset2DAsync(static_cast<uint8_t*>(w->ws.p) + w->o_slot, w->stride, 0, w->stride - w->o_slot,
                             w->n_warps, st));
  CUDA_TRY(cudaMemsetAsync(w->stamps.p, 0, 4ull * w->n_warps, st));
  w->dirty = false;
  return MBE_OK;
}

}  // namespace

extern "C" {

const char* mbe_strerror(int code) {
  switch (code) {
    case MBE_OK: return "ok";
    case MBE_EINVAL: return "invalid argument";
    case MBE_ENOMEM: return "out of memory";
    case MBE_ECUDA: return "CUDA error";
    case MBE_EOVERFLOW: return "frame arena or stack depth exhausted";
    case MBE_ERANGE: return "vertex id out of range";
    case MBE_EDIST: return "multi-GPU claim counter error";
    case MBE_EINTERNAL: return "internal consistency check failed";
    default: return "unknown error";
  }
}

const char* mbe_last_error_detail(void) { return g_detail.c_str(); }

int mbe_load_csr(uint32_t n1, uint32_t n2, const uint64_t* row_ptr, const uint32_t* col_idx, int device,
                 uint32_t flags, mbe_graph** out) {
  const bool dbg = std::getenv("MBE_DEBUG_TIMING") != nullptr;
  auto T = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  load %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - T).count());
    T = n;
  };
  if (flags & ~0xffu) return fail(MBE_EINVAL, "mbe_load_csr flags: only bits 0-7 (ingest threads) are defined");
  g_ingest_threads = flags & 0xffu;
  if (!out) return fail(MBE_EINVAL, "out is NULL");
  *out = nullptr;
  if (!row_ptr && n1) return fail(MBE_EINVAL, "row_ptr is NULL");
  const uint64_t nnz = n1 ? row_ptr[n1] : 0;
  if (n1 && row_ptr[0] != 0) return fail(MBE_EINVAL, "row_ptr[0] != 0");
  for (uint32_t i = 0; i < n1; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return fail(MBE_EINVAL, "row_ptr not monotone at row " + std::to_string(i));
  if (nnz && !col_idx) return fail(MBE_EINVAL, "col_idx is NULL");
  if (nnz >= (1ull << 32)) return fail(MBE_EINVAL, "more than 2^32-1 edges");
  for (uint64_t e = 0; e < nnz; ++e)
    if (col_idx[e] >= n2) {
      uint32_t row = (uint32_t)(std::upper_bound(row_ptr, row_ptr + n1 + 1, e) - row_ptr - 1);
      return fail(MBE_ERANGE, "row " + std::to_string(row) + ": col " + std::to_string(col_idx[e]) +
                                  " >= n2=" + std::to_string(n2));
    }
  lap("validate");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(MBE_ECUDA, "no CUDA device");
  }
  if (device < 0 || device >= ndev) return fail(MBE_EINVAL, "device ordinal out of range");
  CUDA_TRY(cudaSetDevice(device));
  mbe_graph* g = new (std::nothrow) mbe_graph();
  if (!g) return fail(MBE_ENOMEM, "host allocation");
  g->device = device;
  g->n1 = n1;
  g->n2 = n2;
  // row CSR, each row sorted + deduplicated (reading Z8): every thread builds the rows of its range,
  // then the ranges are concatenated at their prefix offsets
  const unsigned nth = ingest_threads(nnz);
  g->off1.assign(n1 + 1, 0);
  {
    std::vector<std::vector<uint32_t>> loc(std::max(1u, nth));
    std::vector<uint32_t> deg(n1);
    std::vector<uint64_t> first(std::max(1u, nth) + 1, 0);  // first row of each thread's range
    parallel_edges(row_ptr, n1, nth, [&](unsigned t, uint64_t a, uint64_t b) {
      first[t] = a;
      if (a >= b) return;
      std::vector<uint32_t>& L = loc[t];
      L.reserve(row_ptr[b] - row_ptr[a]);
      for (uint64_t i = a; i < b; ++i) {
        const size_t s0 = L.size();
        L.insert(L.end(), col_idx + row_ptr[i], col_idx + row_ptr[i + 1]);
        if (!std::is_sorted(L.begin() + s0, L.end())) std::sort(L.begin() + s0, L.end());
        L.erase(std::unique(L.begin() + s0, L.end()), L.end());
        deg[i] = (uint32_t)(L.size() - s0);
      }
    });
    for (uint32_t i = 0; i < n1; ++i) g->off1[i + 1] = g->off1[i] + deg[i];
    g->nE = g->off1[n1];
    g->adj1.resize(g->nE);
    parallel_ranges(std::max(1u, nth), std::max(1u, nth), [&](unsigned, uint64_t a, uint64_t b) {
      for (uint64_t t = a; t < b; ++t) std::copy(loc[t].begin(), loc[t].end(), g->adj1.begin() + g->off1[first[t]]);
    });
  }
  lap("row CSR sort+dedup");
  // column CSR: counting sort with per-thread column counts over row ranges (rows ascending within
  // and across ranges -> every column's rows come out sorted)
  g->off2.assign(n2 + 1, 0);
  g->adj2.resize(g->nE);
  {
    const unsigned T = std::max(1u, std::min(nth, 8u));
    std::vector<uint32_t> cnt((size_t)T * n2, 0);
    parallel_edges(g->off1.data(), n1, T, [&](unsigned t, uint64_t a, uint64_t b) {
      uint32_t* c = cnt.data() + (size_t)t * n2;
      for (uint32_t e = g->off1[a]; e < g->off1[b]; ++e) c[g->adj1[e]]++;
    });
    for (uint32_t j = 0; j < n2; ++j) {
      uint32_t run = g->off2[j];
      for (unsigned t = 0; t < T; ++t) {
        const uint32_t k = cnt[(size_t)t * n2 + j];
        cnt[(size_t)t * n2 + j] = run;
        run += k;
      }
      g->off2[j + 1] = run;
    }
    parallel_edges(g->off1.data(), n1, T, [&](unsigned t, uint64_t a, uint64_t b) {
      uint32_t* c = cnt.data() + (size_t)t * n2;
      for (uint64_t i = a; i < b; ++i)
        for (uint32_t e = g->off1[i]; e < g->off1[i + 1]; ++e) g->adj2[c[g->adj1[e]]++] = (uint32_t)i;
    });
  }
  lap("column CSR");
  if ((g->sm_count = sm_count_of(device)) <= 0) {
    delete g;
    return fail(MBE_ECUDA, "cudaDeviceGetAttribute(multiProcessorCount)");
  }
  lap("device attr + events");
  int side = n2 < n1 ? 2 : 1;
  int rc = build_side(g, side);
  if (rc) {
    delete g;
    return rc;
  }
  lap("build_side (relabel, hv, order, upload)");
  *out = g;
  return MBE_OK;
}

int mbe_get_info(const mbe_graph* g, mbe_graph_info* info) {
  if (!g || !info) return fail(MBE_EINVAL, "NULL argument");
  info->n1 = g->n1;
  info->n2 = g->n2;
  info->n_edges = g->nE;
  uint32_t m1 = 0, m2 = 0;
  for (uint32_t i = 0; i < g->n1; ++i) m1 = std::max(m1, g->off1[i + 1] - g->off1[i]);
  for (uint32_t j = 0; j < g->n2; ++j) m2 = std::max(m2, g->off2[j + 1] - g->off2[j]);
  info->max_deg1 = m1;
  info->max_deg2 = m2;
  info->device = g->device;
  info->h2d_bytes = g->h2d_bytes;
  return MBE_OK;
}

void mbe_free(mbe_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  delete g;
}

int mbe_enumerate(mbe_graph* g, const mbe_config* cfg_in, mbe_result* res, mbe_output* out) {
  auto t0 = std::chrono::steady_clock::now();
  if (!g || !res) return fail(MBE_EINVAL, "NULL graph or result");
  mbe_config cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.struct_size = sizeof(cfg);
  cfg.world = 1;
  if (cfg_in) {
    if (cfg_in->struct_size != sizeof(mbe_config)) return fail(MBE_EINVAL, "mbe_config.struct_size mismatch");
    cfg = *cfg_in;
  }
  if (cfg.world == 0 || cfg.rank >= cfg.world) return fail(MBE_EINVAL, "rank/world");
  if (cfg.threads_per_cta % 32 || cfg.threads_per_cta > MBE_BLOCK)
    return fail(MBE_EINVAL, "threads_per_cta must be a multiple of 32 <= " + std::to_string(MBE_BLOCK));
  if (cfg.bitmap_threshold > 32 * MBE_WMAX) return fail(MBE_EINVAL, "bitmap_threshold > 512");
  if (cfg.candidate_side < 0 || cfg.candidate_side > 2) return fail(MBE_EINVAL, "candidate_side");
  if (cfg.order > 2) return fail(MBE_EINVAL, "order must be MBE_ORDER_ASCENDING, _INPUT or _DESCENDING");
  if (out && (out->cap_records && (!out->rec_off || !out->rec_n1 || !out->rec_n2)))
    return fail(MBE_EINVAL, "mbe_output buffers");
  if (out && out->cap_ids && !out->ids) return fail(MBE_EINVAL, "mbe_output.ids");
  std::memset(res, 0, sizeof(*res));
  CUDA_TRY(cudaSetDevice(g->device));
  const int side = cfg.candidate_side ? cfg.candidate_side : (g->n2 < g->n1 ? 2 : 1);
  int rc = build_side(g, side, cfg.order);
  if (rc) return rc;
  Side& S = g->side[side - 1][cfg.order];
  res->candidate_side = side;
  if (S.nU == 0 || g->nE == 0 || S.n_roots == 0) {
    res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (cfg.per_root) std::memset(cfg.per_root, 0, 32ull * S.nU);
    return MBE_OK;
  }
  const uint32_t threads = cfg.threads_per_cta ? cfg.threads_per_cta : MBE_BLOCK;
  // persistent kernel: every CTA must be co-resident, so clamp to the occupancy limit (cached per handle)
  // instrumented kernel instantiation only when stats / per-root counters / a listing are requested
  const bool instr = (cfg.flags & (MBE_STATS | MBE_NO_RS)) || cfg.per_root || (out && out->cap_records);
  const int smem_warp = instr ? mbe_search_smem_per_warp_instr() : mbe_search_smem_per_warp();
  int& occ = g->occ[instr ? 1 : 0][threads / 32 - 1];
  if (occ <= 0)
    occ = instr ? mbe_search_max_ctas_per_sm_instr((int)threads, smem_warp * (int)(threads / 32))
                : mbe_search_max_ctas_per_sm((int)threads, smem_warp * (int)(threads / 32));
  if (occ <= 0) return fail(MBE_ECUDA, "occupancy query failed for threads_per_cta=" + std::to_string(threads));
  const uint32_t ctas_per_sm = std::min<uint32_t>(cfg.ctas_per_sm ? cfg.ctas_per_sm : (uint32_t)MBE_MINBLOCKS, (uint32_t)occ);
  const uint32_t grid = (uint32_t)g->sm_count * ctas_per_sm;
  const uint32_t n_warps = grid * (threads / 32);
  // auto arena: proportional to the graph, 256 KiB .. 2 MiB per warp (high-water marks: C2 0.32, C3 0.48,
  // C5 0.60, C4 0.91 MB); grown x4 and relaunched on overflow
  const bool grow = cfg.arena_bytes == 0 || (cfg.flags & MBE_ARENA_GROW);
  uint64_t arena = cfg.arena_bytes ? cfg.arena_bytes
                                   : std::min<uint64_t>(2ull << 20, std::max<uint64_t>(256ull << 10, 16ull * (S.nU + S.nV + g->nE)));
  arena = (arena + 255) & ~255ull;
  // auto bit-row threshold: the widest rows (512 columns) whose workspace fits in 80% of free memory
  // (decided once per loaded side; the free-memory query is not repeated on every call)
  uint32_t T = cfg.bitmap_threshold;
  if (!T && S.auto_T) T = S.auto_T;
  if (!T) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    uint64_t pooled = 0;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      for (Workspace* w : g_pool)
        if (!w->busy && w->device == g->device) pooled += w->ws.bytes;
    }
    T = 128;
    for (uint32_t t : {512u, 256u}) {
      if ((double)workspace_stride(S.nU, S.cand, S.maxdegU, arena, mbe_words_for(t)) * n_warps <= 0.8 * (double)(fr + pooled)) {
        T = t;
        break;
      }
    }
    S.auto_T = T;
  }
  const bool auto_T = cfg.bitmap_threshold == 0;
  uint32_t wmax = mbe_words_for(T);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cfg.stream);
  static const bool dbg_timing = std::getenv("MBE_DEBUG_TIMING") != nullptr;
  static const bool dbg_longest = std::getenv("MBE_DEBUG_LONGEST") != nullptr;
  static const bool dbg_hist = std::getenv("MBE_DEBUG_HIST") != nullptr;

  // root twin flags: graph-only, computed once per loaded side (R2 at the root)
  const DevGraph dg = {S.nU, S.nV, g->nE, (const uint32_t*)S.offU.p, (const uint32_t*)S.adjU.p,
                       (const uint32_t*)S.offV.p, (const uint32_t*)S.adjV.p, (const uint64_t*)S.hvU.p,
                       (const uint64_t*)S.hvV.p, (const uint32_t*)S.origUd.p, (const uint32_t*)S.root_order.p,
                       (const uint8_t*)S.twin.p, S.n_roots, S.maxdegU};
  // (twin pruning relies on ascending degrees; the order ablations run without it)
  const bool twin = !(cfg.flags & MBE_NO_TWIN) && cfg.order == 0;
  if (twin && !S.twin_ready) {
    if (mbe_launch_twin(dg, g->sm_count, st) != 0)
      return fail(MBE_ECUDA, std::string("twin kernel launch: ") + cudaGetErrorString(cudaGetLastError()));
    S.twin_ready = true;
  }
  // claim log of a shared-counter call (one entry per claimed chunk, at most one per root)
  if (cfg.claim_counter && g->claim_tab.bytes < 8ull * (S.n_roots + 1)) {
    g->claim_tab.release();
    if (cudaMalloc(&g->claim_tab.p, 8ull * (S.n_roots + 1)) != cudaSuccess) {
      cudaGetLastError();
      return fail(MBE_ENOMEM, "claim log");
    }
    g->claim_tab.bytes = 8ull * (S.n_roots + 1);
  }

  // listing buffers (device) for this call
  struct BufGuard {
    DevBuf rec_off, n1, n2, ids;
    ~BufGuard() {
      for (DevBuf* b : {&rec_off, &n1, &n2, &ids}) b->release();
    }
  } lb;
  const uint64_t cap_rec = out ? out->cap_records : 0, cap_ids = out ? out->cap_ids : 0;
  if (cap_rec) {
    if (cudaMalloc(&lb.rec_off.p, 8 * cap_rec) != cudaSuccess || cudaMalloc(&lb.n1.p, 4 * cap_rec) != cudaSuccess ||
        cudaMalloc(&lb.n2.p, 4 * cap_rec) != cudaSuccess ||
        cudaMalloc(&lb.ids.p, 4 * std::max<uint64_t>(cap_ids, 1)) != cudaSuccess) {
      cudaGetLastError();
      return fail(MBE_ENOMEM, "listing buffers");
    }
  }
  struct WsGuard {
    Workspace* w = nullptr;
    ~WsGuard() {
      if (w) checkin_workspace(w);
    }
  } wg;

  unsigned long long claim_state = 0;  // carried over to a relaunch: replays this call's claimed chunks
  const bool want_stats = instr;
  for (int attempt = 0;; ++attempt) {
    res->attempts = (uint32_t)attempt + 1;
    if (wg.w && wg.w->arena_bytes != arena) {
      checkin_workspace(wg.w);
      wg.w = nullptr;
    }
    const auto tw0 = std::chrono::steady_clock::now();
    if (!wg.w) {
      rc = checkout_workspace(g->device, n_warps, S.nU, S.cand, S.maxdegU, arena, wmax, &wg.w);
      // auto threshold: narrower rows when the device is shared (e.g. several ranks on one GPU)
      while (rc == MBE_ENOMEM && auto_T && T > 128) {
        T /= 2;
        wmax = mbe_words_for(T);
        rc = checkout_workspace(g->device, n_warps, S.nU, S.cand, S.maxdegU, arena, wmax, &wg.w);
      }
      if (rc) return rc;
    }
    Workspace* W = wg.w;
    // a failed launch leaves slots, descriptors and stack tops dirty; a clean one leaves them zero
    if (W->dirty) {
      if ((rc = clear_tables(W, st))) return rc;
      CUDA_TRY(cudaMemsetAsync(W->desc.p, 0, sizeof(Desc) * MBE_MAXDEPTH * n_warps, st));
      CUDA_TRY(cudaMemsetAsync(W->tops.p, 0, 4ull * n_warps, st));
    }
    if (dbg_timing) {
      cudaStreamSynchronize(st);
      std::fprintf(stderr, "  enumerate: workspace checkout + clear %.2f ms (n_warps %u, T %u, arena %llu B, %.1f GB)\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw0).count(), n_warps,
                   T, (unsigned long long)arena, W->ws.bytes / 1e9);
    }
    SearchParams& p = g->sp;
    p.g = dg;
    p.cand_side = side;
    p.T = T;
    p.wide_qcap = MBE_WIDE_QCAP;
    p.wide_ratio = MBE_WIDE_RATIO;
    p.wide_qmax = MBE_WIDE_QMAX;
    p.narrow_qmax = MBE_NARROW_QMAX;
    p.narrow_ratio = MBE_NARROW_RATIO;
    p.ac_min = MBE_AC_MIN;
    p.ac_ratio = MBE_AC_RATIO;
    p.dedup_min = MBE_DEDUP_MIN;
    p.defer_min = cfg.defer_min == 0 ? MBE_DEFER_MIN_DEFAULT : (cfg.defer_min == 0xffffffffu ? 0u : cfg.defer_min);
    p.wide_acmax = MBE_WIDE_ACMAX;
    p.flags = cfg.flags | (twin ? 0u : (uint32_t)MBE_NO_TWIN);
    p.order = cfg.order;
    p.rank = cfg.rank;
    p.world = cfg.world;
    p.claim_counter = reinterpret_cast<unsigned long long*>(cfg.claim_counter);
    p.claim_tab = static_cast<unsigned long long*>(g->claim_tab.p);
    p.gss_div = 4u * cfg.world;
    p.n_warps = n_warps;
    p.watchdog_ns = cfg.watchdog_ms == 0xffffffffu
                        ? 0ull
                        : (unsigned long long)(cfg.watchdog_ms ? cfg.watchdog_ms : MBE_WATCHDOG_MS_DEFAULT) * 1000000ull;
    p.ws = static_cast<uint8_t*>(W->ws.p);
    p.ws_stride = W->stride;
    p.o_slot = W->o_slot;
    p.o_crow = W->o_crow;
    p.o_touched = W->o_touched;
    p.o_lbuf = W->o_lbuf;
    p.o_rbuf = W->o_rbuf;
    p.o_skey = W->o_skey;
    p.o_sval = W->o_sval;
    p.o_pbuf = W->o_pbuf;
    p.o_qbuf = W->o_qbuf;
    p.o_arena = W->o_arena;
    p.skey2_off = W->cap_cand;
    p.arena_words = arena / 4;
    p.desc = static_cast<Desc*>(W->desc.p);
    p.tops = static_cast<unsigned int*>(W->tops.p);
    p.stamps = static_cast<unsigned int*>(W->stamps.p);
    p.hint = static_cast<unsigned int*>(W->hint.p);
    p.gl = static_cast<Globals*>(W->gl.p);
    p.per_root = cfg.per_root ? static_cast<unsigned long long*>(W->per_root.p) : nullptr;
    p.cap_records = cap_rec;
    p.cap_ids = cap_ids;
    p.rec_off = (unsigned long long*)lb.rec_off.p;
    p.rec_n1 = (unsigned int*)lb.n1.p;
    p.rec_n2 = (unsigned int*)lb.n2.p;
    p.out_ids = (unsigned int*)lb.ids.p;

    res->workspace_bytes = W->ws.bytes;
    Globals* dgl = static_cast<Globals*>(W->gl.p);
    CUDA_TRY(cudaMemsetAsync(dgl, 0, want_stats ? sizeof(Globals) : MBE_GLOBALS_HOT_BYTES, st));
    if (want_stats) {
      CUDA_TRY(cudaMemsetAsync(&dgl->t_roots_out, 0xff, 8, st));
      CUDA_TRY(cudaMemsetAsync(&dgl->warp_busy_min, 0xff, 8, st));
    }
    if (claim_state) CUDA_TRY(cudaMemcpyAsync(&dgl->claim_state, &claim_state, 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(W->hint.p, 0, 4ull * ((n_warps + 31) / 32), st));
    if (p.per_root) CUDA_TRY(cudaMemsetAsync(W->per_root.p, 0, 32ull * S.nU, st));
    const int smem = smem_warp * (int)(threads / 32);
    if (!g->ev0) g->ev0 = ev_get(g->device);
    if (!g->ev1) g->ev1 = ev_get(g->device);
    if (!g->ev0 || !g->ev1) return fail(MBE_ECUDA, "cudaEventCreate");
    const int lrc = instr ? mbe_launch_search_instr(p, (int)grid, (int)threads, smem, st, g->ev0, g->ev1)
                          : mbe_launch_search(p, (int)grid, (int)threads, smem, st, g->ev0, g->ev1);
    if (lrc != 0)
      return fail(MBE_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(cudaGetLastError()));
    Globals hg;
    CUDA_TRY(cudaMemcpyAsync(&hg, dgl, want_stats ? sizeof(Globals) : MBE_GLOBALS_HOT_BYTES, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    W->dirty = hg.error != 0;  // slots may hold partial counts, frames may be left on the stacks
    if (hg.error) {
      if ((hg.error == 1u) && grow && attempt < 6) {
        arena *= 4;  // grow and relaunch; a shared-counter call replays exactly the chunks it claimed
        claim_state = hg.claim_state;
        continue;
      }
      if (hg.error == 4u)
        return fail(MBE_EINTERNAL, "device watchdog: no task completed for " +
                                       std::to_string(p.watchdog_ns / 1000000ull) + " ms (mbe_config.watchdog_ms)");
      if (hg.error == 3u)
        return fail(MBE_EINTERNAL, "device consistency check failed (info " + std::to_string(hg.err_info) + ")");
      return fail(MBE_EOVERFLOW, hg.error == 2u ? "stack depth > " + std::to_string(MBE_MAXDEPTH)
                                                : "frame arena exhausted (arena_bytes=" + std::to_string(arena) + ")");
    }
    res->count = hg.count;
    res->hash = hg.hash;
    res->tasks = hg.tasks;
    res->pruned = hg.pruned;
    res->steals = hg.steals;
    res->kernel_ms = ms;
    res->n_warps = n_warps;
    res->roots_claimed = hg.roots_run;
    res->claim_chunks = cfg.claim_counter ? (uint32_t)(hg.claim_state >> 33) : 0u;
    if (want_stats) {
      res->alg_bytes = hg.alg_bytes;
      res->alg_bytes_list = hg.alg_list;
      res->alg_bytes_bitrow = hg.alg_bitrow;
      res->alg_bytes_write = hg.alg_write;
      res->list_tasks = hg.list_tasks;
      res->bitmap_tasks = hg.bitmap_tasks;
      res->frames = hg.frames;
      res->max_depth = hg.max_depth;
      for (int k = 0; k < 16; ++k) res->phase_cycles[k] = hg.phase[k];
      for (int k = 0; k < 3; ++k) res->max_task_cycles[k] = hg.max_task[k];
      for (int k = 0; k < 16; ++k) res->max_phase_cycles[k] = hg.max_phase[k];
      res->roots_out_ms = hg.t_roots_out == ~0ull ? -1.0 : (double)hg.t_roots_out * 1e-6;
      int clk_khz = 0;
      cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, g->device);
      const double cyc_per_ms = clk_khz > 0 ? (double)clk_khz : 1.965e6;
      for (int b = 0; b < 20; ++b) res->busy_hist[b] = (uint32_t)hg.warp_busy_hist[b];
      res->busy_ms_min = hg.warp_busy_min == ~0ull ? 0.0 : (double)hg.warp_busy_min / cyc_per_ms;
      res->busy_ms_max = (double)hg.warp_busy_max / cyc_per_ms;
      res->busy_ms_mean = (double)hg.warp_busy_sum / cyc_per_ms / (double)n_warps;
    } else {
      res->roots_out_ms = -1.0;
    }
    if (dbg_longest && (cfg.flags & MBE_STATS)) {
      const unsigned long long* L = hg.longest;
      std::fprintf(stderr,
                   "longest list task: %.3f ms root=%llu x=%llu deg=%llu |L'|=%llu touched=%llu |P'|=%llu |Q'|=%llu "
                   "Wchild=%llu kept=%llu nP=%llu | isect %.3f scan %.3f classify %.3f sort %.3f child %.3f ms "
                   "(before dedup %.3f ms, dedup %.3f ms -> %llu rows, antichain %.3f ms, prune %.3f ms = meta %.3f + eq %.3f + Q %.3f)\n",
                   L[0] / 1.965e6, L[1], L[2], L[3], L[4], L[5], L[6], L[7], L[8], L[14], L[15], L[9] / 1.965e6,
                   L[10] / 1.965e6, L[11] / 1.965e6, L[12] / 1.965e6, L[13] / 1.965e6, L[20] / 1.965e6, L[16] / 1.965e6, L[18],
                   L[17] / 1.965e6, L[19] / 1.965e6, L[21] / 1.965e6, L[22] / 1.965e6, L[23] / 1.965e6);
    }
    if (dbg_hist && (cfg.flags & MBE_STATS)) {
      for (int b = 0; b < 24; ++b)
        if (hg.hist[0][b])
          std::fprintf(stderr, "bit-row tasks |P|+|Q| in [%d,%d): %llu tasks, %.3f ms warp time, %.2f us/task\n",
                       (1 << b) - 1, (2 << b) - 1, hg.hist[0][b], hg.hist[1][b] / 1.965e6,
                       hg.hist[1][b] / 1.965e3 / (double)hg.hist[0][b]);
      std::fprintf(stderr, "warps first idle / exiting per 2 ms:");
      for (int b = 0; b < 64; ++b)
        if (hg.busy_hist[b] || hg.exit_hist[b]) std::fprintf(stderr, " [%d] %llu/%llu", 2 * b, hg.busy_hist[b], hg.exit_hist[b]);
      std::fprintf(stderr, "\n");
      for (int k = 0; k < 4; ++k) {
        std::fprintf(stderr, "%s warp-ms by completion time (2 ms buckets):",
                     k == 0 ? "root task" : (k == 1 ? "list task" : (k == 2 ? "bitrow task" : "failed steal")));
        for (int b = 0; b < 64; ++b)
          if (hg.tl_hist[k][b]) std::fprintf(stderr, " [%d] %.0f", 2 * b, hg.tl_hist[k][b] / 1.965e6);
        std::fprintf(stderr, "\n");
      }
      const char* sub[3] = {"compress", "prune", "antichain"};
      for (int b = 29; b < 32; ++b)
        if (hg.hist[0][b])
          std::fprintf(stderr, "wide child build, %s: %llu calls, %.3f ms warp time, %.2f us/call\n", sub[b - 29],
                       hg.hist[0][b], hg.hist[1][b] / 1.965e6, hg.hist[1][b] / 1.965e3 / (double)hg.hist[0][b]);
      std::fprintf(stderr, "max arena words per warp: %llu (%.2f MB)\n", hg.max_arena_words, hg.max_arena_words * 4e-6);
      for (int b = 0; b < 12; ++b)
        if (hg.list_nt_hist[0][b])
          std::fprintf(stderr, "list tasks touched in [4^%d, 4^%d): %llu tasks, %.3f ms warp time\n", b, b + 1,
                       hg.list_nt_hist[0][b], hg.list_nt_hist[1][b] / 1.965e6);
      for (int k = 0; k < 2; ++k)
        for (int b = 0; b < 8; ++b)
          if (hg.wide_hist[2 * k][b])
            std::fprintf(stderr, "wide tasks %s in [4^%d, 4^%d): %llu tasks, %.3f ms warp time\n", k ? "|P|" : "|Q|", b,
                         b + 1, hg.wide_hist[2 * k][b], hg.wide_hist[2 * k + 1][b] / 1.965e6);
      for (int b = 24; b < 29; ++b)
        if (hg.hist[0][b])
          std::fprintf(stderr, "bit-row tasks W=%d: %llu tasks, %.3f ms warp time, %.2f us/task\n", 1 << (b - 24),
                       hg.hist[0][b], hg.hist[1][b] / 1.965e6, hg.hist[1][b] / 1.965e3 / (double)hg.hist[0][b]);
    }
    if (cfg.per_root) {
      std::vector<uint64_t> pr(4ull * S.nU);
      CUDA_TRY(cudaMemcpy(pr.data(), W->per_root.p, 32ull * S.nU, cudaMemcpyDeviceToHost));
      for (uint32_t r = 0; r < S.nU; ++r) std::memcpy(cfg.per_root + 4ull * S.origU[r], pr.data() + 4ull * r, 32);
    }
    if (cap_rec) {
      uint64_t nrec = std::min<uint64_t>(hg.out_records, cap_rec);
      std::vector<uint64_t> ro(nrec);
      std::vector<uint32_t> a(nrec), b(nrec);
      if (nrec) {
        CUDA_TRY(cudaMemcpy(ro.data(), lb.rec_off.p, 8 * nrec, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(a.data(), lb.n1.p, 4 * nrec, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(b.data(), lb.n2.p, 4 * nrec, cudaMemcpyDeviceToHost));
      }
      // keep only records whose ids fit entirely
      uint64_t written = 0;
      for (uint64_t r = 0; r < nrec; ++r) {
        if (ro[r] == ~0ull || ro[r] + a[r] + b[r] > cap_ids) continue;
        out->rec_off[written] = ro[r];
        out->rec_n1[written] = a[r];
        out->rec_n2[written] = b[r];
        ++written;
      }
      uint64_t nid = std::min<uint64_t>(hg.out_ids, cap_ids);
      if (nid) CUDA_TRY(cudaMemcpy(out->ids, lb.ids.p, 4 * nid, cudaMemcpyDeviceToHost));
      for (uint64_t r = 0; r < written; ++r) {  // canonical order inside each side
        std::sort(out->ids + out->rec_off[r], out->ids + out->rec_off[r] + out->rec_n1[r]);
        std::sort(out->ids + out->rec_off[r] + out->rec_n1[r],
                  out->ids + out->rec_off[r] + out->rec_n1[r] + out->rec_n2[r]);
      }
      res->records_written = written;
      res->truncated = written < hg.count ? 1u : 0u;
    }
    break;
  }
  res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return MBE_OK;
}

// ------------------------------------------------------------------ cross-process claim counter
struct mbe_counter {
  int device = 0;
  bool owner = false;  // created here (cudaFree) vs opened from a handle (cudaIpcCloseMemHandle)
  void* p = nullptr;
};

int mbe_counter_create(int device, mbe_counter** out) {
  if (!out) return fail(MBE_EINVAL, "out is NULL");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  mbe_counter* c = new (std::nothrow) mbe_counter();
  if (!c) return fail(MBE_ENOMEM, "host allocation");
  c->device = device;
  c->owner = true;
  if (cudaMalloc(&c->p, 256) != cudaSuccess || cudaMemset(c->p, 0, 256) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    if (c->p) cudaFree(c->p);
    delete c;
    return fail(MBE_ECUDA, "claim counter allocation");
  }
  *out = c;
  return MBE_OK;
}

int mbe_counter_ipc_handle(const mbe_counter* c, void* handle) {
  if (!c || !handle) return fail(MBE_EINVAL, "NULL argument");
  if (!c->owner) return fail(MBE_EINVAL, "only the creating process exports the handle");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle is 64 bytes");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->p));
  std::memcpy(handle, &h, 64);
  return MBE_OK;
}

int mbe_counter_open(int device, const void* handle, mbe_counter** out) {
  if (!handle || !out) return fail(MBE_EINVAL, "NULL argument");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  mbe_counter* c = new (std::nothrow) mbe_counter();
  if (!c) return fail(MBE_ENOMEM, "host allocation");
  c->device = device;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  const cudaError_t e = cudaIpcOpenMemHandle(&c->p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return fail(e == cudaErrorDeviceUninitialized ? MBE_EDIST : MBE_ECUDA,
                std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  }
  *out = c;
  return MBE_OK;
}

uint64_t* mbe_counter_ptr(const mbe_counter* c) { return c ? static_cast<uint64_t*>(c->p) : nullptr; }

int mbe_counter_reset(mbe_counter* c, void* stream) {
  if (!c) return fail(MBE_EINVAL, "NULL counter");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaMemsetAsync(c->p, 0, 8, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MBE_OK;
}

uint64_t mbe_counter_read(mbe_counter* c) {
  if (!c) return 0;
  uint64_t v = 0;
  cudaSetDevice(c->device);
  if (cudaMemcpy(&v, c->p, 8, cudaMemcpyDeviceToHost) != cudaSuccess) cudaGetLastError();
  return v;
}

void mbe_counter_close(mbe_counter* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->owner) cudaFree(c->p);
  else cudaIpcCloseMemHandle(c->p);
  delete c;
}

void mbe_release_workspaces(void) {
  {
    std::lock_guard<std::mutex> lk(g_graph_cache_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    for (const CachedBlock& c : g_graph_cache) {
      cudaSetDevice(c.device);
      cudaFree(c.p);
    }
    g_graph_cache.clear();
    cudaSetDevice(dev);
  }
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto it = g_pool.begin(); it != g_pool.end();) {
    if (!(*it)->busy) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaSetDevice((*it)->device);
      (*it)->release();
      cudaSetDevice(dev);
      delete *it;
      it = g_pool.erase(it);
    } else {
      ++it;
    }
  }
}

// Canonical listing text: host post-processing of the
// records mbe_enumerate wrote, so that listings of different configurations diff byte-exactly.
int mbe_format_listing(const mbe_output* out, uint64_t n_records, char* buf, uint64_t cap, uint64_t* needed) {
  if (!out || !needed) return fail(MBE_EINVAL, "out or needed is NULL");
  if (n_records > out->cap_records) return fail(MBE_EINVAL, "n_records > cap_records");
  if (n_records && (!out->rec_off || !out->rec_n1 || !out->rec_n2 || !out->ids))
    return fail(MBE_EINVAL, "mbe_output buffer is NULL");
  if (cap && !buf) return fail(MBE_EINVAL, "buf is NULL with cap > 0");
  std::vector<std::string> lines;
  try {
    lines.resize(n_records);
    for (uint64_t r = 0; r < n_records; ++r) {
      const uint64_t o = out->rec_off[r], a = out->rec_n1[r], b = out->rec_n2[r];
      if (o > out->cap_ids || a + b > out->cap_ids - o)
        return fail(MBE_EINVAL, "record " + std::to_string(r) + " lies outside ids[cap_ids]");
      std::string& s = lines[r];
      s.reserve(8 + 8 * (a + b));
      s += "L: ";
      for (uint64_t i = 0; i < a; ++i) {
        if (i) s += ',';
        s += std::to_string(out->ids[o + i]);
      }
      s += " | R: ";
      for (uint64_t i = 0; i < b; ++i) {
        if (i) s += ',';
        s += std::to_string(out->ids[o + a + i]);
      }
      s += '\n';
    }
    std::sort(lines.begin(), lines.end());  // byte order (std::string compares as unsigned char)
  } catch (const std::bad_alloc&) {
    return fail(MBE_ENOMEM, "listing text");
  }
  uint64_t total = 0;
  for (const auto& s : lines) total += s.size();
  *needed = total;
  if (cap < total) return fail(MBE_EOVERFLOW, "listing text needs " + std::to_string(total) + " bytes");
  uint64_t pos = 0;
  for (const auto& s : lines) {
    std::memcpy(buf + pos, s.data(), s.size());
    pos += s.size();
  }
  return MBE_OK;
}

}  // extern "C"
