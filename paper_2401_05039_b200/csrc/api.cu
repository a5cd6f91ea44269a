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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
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

template <class T>
int upload(DevBuf& b, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) return fail(MBE_ENOMEM, "cudaMalloc graph");
  b.bytes = bytes;
  if (!v.empty()) CUDA_TRY(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return MBE_OK;
}

struct Side {
  bool built = false;
  uint32_t nU = 0, nV = 0, n_roots = 0, maxdegU = 0;
  std::vector<uint32_t> origU;  // host copy: rank -> original id
  std::vector<uint32_t> rankU;  // host copy: original id -> rank
  DevBuf offU, adjU, offV, adjV, hvU, hvV, origUd, root_order, twin;
  void release() {
    for (DevBuf* b : {&offU, &adjU, &offV, &adjV, &hvU, &hvV, &origUd, &root_order, &twin}) b->release();
    built = false;
  }
};

}  // namespace

struct mbe_graph {
  int device = 0;
  uint32_t n1 = 0, n2 = 0;
  uint64_t nE = 0;
  // deduplicated host CSR in both directions (original ids)
  std::vector<uint32_t> off1, adj1, off2, adj2;
  Side side[2];
  // workspace cache
  DevBuf ws, desc, tops, stamps, hint, gl, per_root;
  uint64_t ws_stride = 0, arena_bytes = 0;
  uint32_t ws_warps = 0, ws_side = 0, ws_wmax = 0;
  bool ws_dirty = true;
  SearchParams sp;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int sm_count = 0;
  ~mbe_graph() {
    for (auto& s : side) s.release();
    for (DevBuf* b : {&ws, &desc, &tops, &stamps, &hint, &gl, &per_root}) b->release();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
};

namespace {

// Build the device graph for candidate side s (1 = rows, 2 = cols).
int build_side(mbe_graph* g, int s) {
  Side& S = g->side[s - 1];
  if (S.built) return MBE_OK;
  const std::vector<uint32_t>& offC = s == 1 ? g->off1 : g->off2;  // candidate side CSR
  const std::vector<uint32_t>& adjC = s == 1 ? g->adj1 : g->adj2;
  const uint32_t nU = s == 1 ? g->n1 : g->n2, nV = s == 1 ? g->n2 : g->n1;
  S.nU = nU;
  S.nV = nV;
  // rank by ascending (degree, original id): counting sort over degrees (stable in id)
  uint32_t maxdeg = 0;
  for (uint32_t u = 0; u < nU; ++u) maxdeg = std::max(maxdeg, offC[u + 1] - offC[u]);
  std::vector<uint32_t> bucket(maxdeg + 2, 0);
  for (uint32_t u = 0; u < nU; ++u) bucket[offC[u + 1] - offC[u] + 1]++;
  for (uint32_t d = 1; d < bucket.size(); ++d) bucket[d] += bucket[d - 1];
  S.origU.assign(nU, 0);
  S.rankU.assign(nU, 0);
  for (uint32_t u = 0; u < nU; ++u) {
    uint32_t r = bucket[offC[u + 1] - offC[u]]++;
    S.origU[r] = u;
    S.rankU[u] = r;
  }
  S.maxdegU = maxdeg;
  // adjU[rank] = sorted V ids; adjV[v] = sorted ranks
  std::vector<uint32_t> offU(nU + 1, 0), adjU(g->nE), offV(nV + 1, 0), adjV(g->nE);
  for (uint32_t r = 0; r < nU; ++r) {
    uint32_t u = S.origU[r];
    offU[r + 1] = offU[r] + (offC[u + 1] - offC[u]);
    std::copy(adjC.begin() + offC[u], adjC.begin() + offC[u + 1], adjU.begin() + offU[r]);
  }
  for (uint64_t e = 0; e < g->nE; ++e) offV[adjU[e] + 1]++;
  for (uint32_t v = 0; v < nV; ++v) offV[v + 1] += offV[v];
  {
    std::vector<uint32_t> fill(offV.begin(), offV.end() - 1);
    for (uint32_t r = 0; r < nU; ++r)
      for (uint32_t e = offU[r]; e < offU[r + 1]; ++e) adjV[fill[adjU[e]]++] = r;
  }
  // hash terms: side bit 0 for side 1 (rows), 1 for side 2 (cols)
  std::vector<uint64_t> hvU(nU), hvV(nV);
  const uint64_t bu = s == 1 ? 0 : 1, bv = 1 - bu;
  for (uint32_t r = 0; r < nU; ++r) hvU[r] = mbe_mix64(2ull * S.origU[r] + bu);
  for (uint32_t v = 0; v < nV; ++v) hvV[v] = mbe_mix64(2ull * v + bv);
  // execution order of level-1 subtrees: descending P-role 2-hop estimate
  //   cost(x) = Σ_{u ∈ N(x)} |{w ∈ N(u) : w > x}|, ties by rank
  std::vector<std::pair<uint64_t, uint32_t>> cost;
  cost.reserve(nU);
  for (uint32_t r = 0; r < nU; ++r) {
    if (offU[r + 1] == offU[r]) continue;
    uint64_t c = 0;
    for (uint32_t e = offU[r]; e < offU[r + 1]; ++e) {
      uint32_t u = adjU[e];
      const uint32_t* b = adjV.data() + offV[u];
      const uint32_t* en = adjV.data() + offV[u + 1];
      c += (uint64_t)(en - std::upper_bound(b, en, r));
    }
    cost.push_back({c, r});
  }
  std::sort(cost.begin(), cost.end(), [](const std::pair<uint64_t, uint32_t>& a, const std::pair<uint64_t, uint32_t>& b) {
    if (a.first != b.first) return a.first > b.first;
    return a.second < b.second;
  });
  std::vector<uint32_t> order(cost.size());
  for (size_t k = 0; k < cost.size(); ++k) order[k] = cost[k].second;
  S.n_roots = (uint32_t)order.size();
  int rc;
  if ((rc = upload(S.offU, offU)) || (rc = upload(S.adjU, adjU)) || (rc = upload(S.offV, offV)) ||
      (rc = upload(S.adjV, adjV)) || (rc = upload(S.hvU, hvU)) || (rc = upload(S.hvV, hvV)) ||
      (rc = upload(S.origUd, S.origU)) || (rc = upload(S.root_order, order))) {
    S.release();
    return rc;
  }
  if (cudaMalloc(&S.twin.p, std::max<size_t>(nU, 16)) != cudaSuccess) {
    S.release();
    return fail(MBE_ENOMEM, "cudaMalloc twin");
  }
  S.built = true;
  return MBE_OK;
}

uint64_t align256(uint64_t x) { return (x + 255) & ~255ull; }

int ensure_workspace(mbe_graph* g, int s, uint32_t n_warps, uint64_t arena_bytes, uint32_t wmax) {
  Side& S = g->side[s - 1];
  if (g->ws.p && g->ws_warps == n_warps && g->ws_side == (uint32_t)s && g->arena_bytes == arena_bytes &&
      g->ws_wmax == wmax) {
    return MBE_OK;
  }
  for (DevBuf* b : {&g->ws, &g->desc, &g->tops, &g->stamps, &g->hint, &g->per_root}) b->release();
  const uint64_t nU = std::max<uint32_t>(S.nU, 1);
  SearchParams& p = g->sp;
  uint64_t o = 0;
  p.o_slot = o; o = align256(o + nU * 32);
  p.o_touched = o; o = align256(o + nU * 4);
  p.o_lbuf = o; o = align256(o + (uint64_t)std::max<uint32_t>(S.maxdegU, 32 * MBE_WMAX) * 4);
  p.o_rbuf = o; o = align256(o + nU * 4);
  p.o_skey = o; o = align256(o + nU * 16);
  p.o_sval = o; o = align256(o + nU * 8);
  p.o_pbuf = o; o = align256(o + nU * wmax * 4);
  p.o_qbuf = o; o = align256(o + nU * wmax * 4);
  p.o_arena = o; o = align256(o + arena_bytes);
  g->ws_stride = o;
  const uint64_t total = o * n_warps;
  if (cudaMalloc(&g->ws.p, total) != cudaSuccess) {
    cudaGetLastError();
    return fail(MBE_ENOMEM, "workspace of " + std::to_string(total >> 20) + " MiB (" + std::to_string(n_warps) +
                                " warps): reduce ctas_per_sm/threads_per_cta/arena_bytes");
  }
  g->ws.bytes = total;
  if (cudaMalloc(&g->desc.p, sizeof(Desc) * MBE_MAXDEPTH * n_warps) != cudaSuccess ||
      cudaMalloc(&g->tops.p, 4ull * n_warps) != cudaSuccess || cudaMalloc(&g->stamps.p, 4ull * n_warps) != cudaSuccess ||
      cudaMalloc(&g->hint.p, 4ull * ((n_warps + 31) / 32)) != cudaSuccess ||
      cudaMalloc(&g->per_root.p, 32ull * nU) != cudaSuccess) {
    cudaGetLastError();
    return fail(MBE_ENOMEM, "workspace descriptors");
  }
  CUDA_TRY(cudaMemset(g->stamps.p, 0, 4ull * n_warps));
  g->ws_warps = n_warps;
  g->ws_side = s;
  g->arena_bytes = arena_bytes;
  g->ws_wmax = wmax;
  g->ws_dirty = true;  // counters/bits/tags must be zeroed before use
  return MBE_OK;
}

// zero the per-warp cnt/bits/tag tables (required invariant: zero between tasks)
int clear_tables(mbe_graph* g, cudaStream_t st) {
  const SearchParams& p = g->sp;
  // per-vertex slots (count, tag, bit row) must be zero between tasks
  CUDA_TRY(cudaMemset2DAsync(static_cast<uint8_t*>(g->ws.p) + p.o_slot, g->ws_stride, 0, p.o_touched - p.o_slot,
                             g->ws_warps, st));
  CUDA_TRY(cudaMemsetAsync(g->stamps.p, 0, 4ull * g->ws_warps, st));
  g->ws_dirty = false;
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
  (void)flags;
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
  // row CSR, each row sorted + deduplicated (reading Z8)
  g->off1.assign(n1 + 1, 0);
  g->adj1.reserve(nnz);
  for (uint32_t i = 0; i < n1; ++i) {
    size_t b = g->adj1.size();
    g->adj1.insert(g->adj1.end(), col_idx + row_ptr[i], col_idx + row_ptr[i + 1]);
    std::sort(g->adj1.begin() + b, g->adj1.end());
    g->adj1.erase(std::unique(g->adj1.begin() + b, g->adj1.end()), g->adj1.end());
    g->off1[i + 1] = (uint32_t)g->adj1.size();
  }
  g->nE = g->adj1.size();
  // column CSR (counting sort; rows visited ascending -> sorted)
  g->off2.assign(n2 + 1, 0);
  g->adj2.resize(g->nE);
  for (uint32_t c : g->adj1) g->off2[c + 1]++;
  for (uint32_t j = 0; j < n2; ++j) g->off2[j + 1] += g->off2[j];
  {
    std::vector<uint32_t> fill(g->off2.begin(), g->off2.end() - 1);
    for (uint32_t i = 0; i < n1; ++i)
      for (uint32_t e = g->off1[i]; e < g->off1[i + 1]; ++e) g->adj2[fill[g->adj1[e]]++] = i;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    delete g;
    return fail(MBE_ECUDA, "cudaGetDeviceProperties");
  }
  g->sm_count = prop.multiProcessorCount;
  if (cudaEventCreate(&g->ev0) != cudaSuccess || cudaEventCreate(&g->ev1) != cudaSuccess) {
    delete g;
    return fail(MBE_ECUDA, "cudaEventCreate");
  }
  int side = n2 < n1 ? 2 : 1;
  int rc = build_side(g, side);
  if (rc) {
    delete g;
    return rc;
  }
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
  if (cfg.threads_per_cta % 32 || cfg.threads_per_cta > 256) return fail(MBE_EINVAL, "threads_per_cta must be a multiple of 32 <= 256");
  if (cfg.bitmap_threshold > 32 * MBE_WMAX) return fail(MBE_EINVAL, "bitmap_threshold > 128");
  if (cfg.candidate_side < 0 || cfg.candidate_side > 2) return fail(MBE_EINVAL, "candidate_side");
  if (out && (out->cap_records && (!out->rec_off || !out->rec_n1 || !out->rec_n2)))
    return fail(MBE_EINVAL, "mbe_output buffers");
  if (out && out->cap_ids && !out->ids) return fail(MBE_EINVAL, "mbe_output.ids");
  std::memset(res, 0, sizeof(*res));
  CUDA_TRY(cudaSetDevice(g->device));
  const int side = cfg.candidate_side ? cfg.candidate_side : (g->n2 < g->n1 ? 2 : 1);
  int rc = build_side(g, side);
  if (rc) return rc;
  Side& S = g->side[side - 1];
  res->candidate_side = side;
  if (S.nU == 0 || g->nE == 0 || S.n_roots == 0) {
    res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (cfg.per_root) std::memset(cfg.per_root, 0, 32ull * S.nU);
    return MBE_OK;
  }
  const uint32_t threads = cfg.threads_per_cta ? cfg.threads_per_cta : 256;
  const uint32_t ctas_per_sm = cfg.ctas_per_sm ? cfg.ctas_per_sm : 2;
  const uint32_t T = cfg.bitmap_threshold ? cfg.bitmap_threshold : 128;
  const uint32_t wmax = mbe_words_for(T);
  const uint32_t grid = (uint32_t)g->sm_count * ctas_per_sm;
  const uint32_t n_warps = grid * (threads / 32);
  // auto arena: proportional to the graph, 256 KiB .. 8 MiB per warp; grown x4 and retried on overflow
  uint64_t arena = cfg.arena_bytes ? cfg.arena_bytes
                                   : std::min<uint64_t>(8ull << 20, std::max<uint64_t>(256ull << 10, 16ull * (S.nU + S.nV + g->nE)));
  arena = (arena + 255) & ~255ull;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cfg.stream);

  // listing buffers (device) for this call
  DevBuf d_rec_off, d_n1, d_n2, d_ids;
  const uint64_t cap_rec = out ? out->cap_records : 0, cap_ids = out ? out->cap_ids : 0;
  if (cap_rec) {
    if (cudaMalloc(&d_rec_off.p, 8 * cap_rec) != cudaSuccess || cudaMalloc(&d_n1.p, 4 * cap_rec) != cudaSuccess ||
        cudaMalloc(&d_n2.p, 4 * cap_rec) != cudaSuccess || cudaMalloc(&d_ids.p, 4 * std::max<uint64_t>(cap_ids, 1)) != cudaSuccess) {
      cudaGetLastError();
      for (DevBuf* b : {&d_rec_off, &d_n1, &d_n2, &d_ids}) b->release();
      return fail(MBE_ENOMEM, "listing buffers");
    }
  }
  if (!g->gl.p && cudaMalloc(&g->gl.p, sizeof(Globals)) != cudaSuccess) return fail(MBE_ENOMEM, "globals");

  int result = MBE_OK;
  for (int attempt = 0;; ++attempt) {
    rc = ensure_workspace(g, side, n_warps, arena, wmax);
    if (rc) { result = rc; break; }
    if (g->ws_dirty && (rc = clear_tables(g, st))) { result = rc; break; }
    SearchParams& p = g->sp;
    p.g.nU = S.nU;
    p.g.nV = S.nV;
    p.g.nE = g->nE;
    p.g.offU = (const uint32_t*)S.offU.p;
    p.g.adjU = (const uint32_t*)S.adjU.p;
    p.g.offV = (const uint32_t*)S.offV.p;
    p.g.adjV = (const uint32_t*)S.adjV.p;
    p.g.hvU = (const uint64_t*)S.hvU.p;
    p.g.hvV = (const uint64_t*)S.hvV.p;
    p.g.origU = (const uint32_t*)S.origUd.p;
    p.g.root_order = (const uint32_t*)S.root_order.p;
    p.g.twin = (const uint8_t*)S.twin.p;
    p.g.n_roots = S.n_roots;
    p.g.maxdegU = S.maxdegU;
    p.cand_side = side;
    p.T = T;
    p.flags = cfg.flags;
    p.rank = cfg.rank;
    p.world = cfg.world;
    p.claim_counter = reinterpret_cast<unsigned long long*>(cfg.claim_counter);
    p.n_warps = n_warps;
    {
      const char* wd = std::getenv("MBE_WATCHDOG_MS");
      p.watchdog_ns = (wd ? std::strtoull(wd, nullptr, 10) : 120000ull) * 1000000ull;
    }
    p.ws = static_cast<uint8_t*>(g->ws.p);
    p.ws_stride = g->ws_stride;
    p.arena_words = arena / 4;
    p.desc = static_cast<Desc*>(g->desc.p);
    p.tops = static_cast<unsigned int*>(g->tops.p);
    p.stamps = static_cast<unsigned int*>(g->stamps.p);
    p.hint = static_cast<unsigned int*>(g->hint.p);
    p.gl = static_cast<Globals*>(g->gl.p);
    p.per_root = cfg.per_root ? static_cast<unsigned long long*>(g->per_root.p) : nullptr;
    p.cap_records = cap_rec;
    p.cap_ids = cap_ids;
    p.rec_off = (unsigned long long*)d_rec_off.p;
    p.rec_n1 = (unsigned int*)d_n1.p;
    p.rec_n2 = (unsigned int*)d_n2.p;
    p.out_ids = (unsigned int*)d_ids.p;

    CUDA_TRY(cudaMemsetAsync(g->gl.p, 0, sizeof(Globals), st));
    CUDA_TRY(cudaMemsetAsync(g->desc.p, 0, sizeof(Desc) * MBE_MAXDEPTH * n_warps, st));
    CUDA_TRY(cudaMemsetAsync(g->tops.p, 0, 4ull * n_warps, st));
    CUDA_TRY(cudaMemsetAsync(g->hint.p, 0, 4ull * ((n_warps + 31) / 32), st));
    if (p.per_root) CUDA_TRY(cudaMemsetAsync(g->per_root.p, 0, 32ull * S.nU, st));
    const int smem = mbe_search_smem_per_warp() * (int)(threads / 32);
    CUDA_TRY(cudaEventRecord(g->ev0, st));
    if (mbe_launch_search(p, (int)grid, (int)threads, smem, st) != 0) {
      result = fail(MBE_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(cudaGetLastError()));
      break;
    }
    CUDA_TRY(cudaEventRecord(g->ev1, st));
    Globals hg;
    CUDA_TRY(cudaMemcpyAsync(&hg, g->gl.p, sizeof(Globals), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    if (hg.error) {
      g->ws_dirty = true;  // tables may hold partial counts
      if ((hg.error == 1u) && !cfg.arena_bytes && attempt < 6) {
        arena *= 4;  // auto arena: grow and retry
        continue;
      }
      if (hg.error == 4u) {
        result = fail(MBE_EINTERNAL, "device watchdog expired (MBE_WATCHDOG_MS)");
      } else if (hg.error == 3u) {
        result = fail(MBE_EINTERNAL, "device consistency check failed (info " + std::to_string(hg.err_info) + ")");
      } else {
        result = fail(MBE_EOVERFLOW, hg.error == 2u ? "stack depth > " + std::to_string(MBE_MAXDEPTH)
                                                    : "frame arena exhausted (arena_bytes=" + std::to_string(arena) + ")");
      }
      break;
    }
    res->count = hg.count;
    res->hash = hg.hash;
    res->tasks = hg.tasks;
    res->pruned = hg.pruned;
    res->steals = hg.steals;
    res->kernel_ms = ms;
    res->alg_bytes = hg.alg_bytes;
    res->list_tasks = hg.list_tasks;
    res->bitmap_tasks = hg.bitmap_tasks;
    res->frames = hg.frames;
    res->n_warps = n_warps;
    res->max_depth = hg.max_depth;
    for (int k = 0; k < 8; ++k) res->phase_cycles[k] = hg.phase[k];
    if (cfg.per_root) {
      std::vector<uint64_t> pr(4ull * S.nU);
      CUDA_TRY(cudaMemcpy(pr.data(), g->per_root.p, 32ull * S.nU, cudaMemcpyDeviceToHost));
      for (uint32_t r = 0; r < S.nU; ++r)
        std::memcpy(cfg.per_root + 4ull * S.origU[r], pr.data() + 4ull * r, 32);
    }
    if (cap_rec) {
      uint64_t nrec = std::min<uint64_t>(hg.out_records, cap_rec);
      std::vector<uint64_t> ro(nrec);
      std::vector<uint32_t> a(nrec), b(nrec);
      if (nrec) {
        CUDA_TRY(cudaMemcpy(ro.data(), d_rec_off.p, 8 * nrec, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(a.data(), d_n1.p, 4 * nrec, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(b.data(), d_n2.p, 4 * nrec, cudaMemcpyDeviceToHost));
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
      if (nid) CUDA_TRY(cudaMemcpy(out->ids, d_ids.p, 4 * nid, cudaMemcpyDeviceToHost));
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
  for (DevBuf* b : {&d_rec_off, &d_n1, &d_n2, &d_ids}) b->release();
  res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

}  // extern "C"
