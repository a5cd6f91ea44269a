// search.cu — persistent MBEA search kernel for sm_100a.
//
// One WARP is one search worker ("warps = sibling tasks"): it
// owns a LIFO stack of immutable frames in an HBM arena, claims level-1
// subtrees (root tasks) from a global cursor, and steals single tasks from
// other warps' frames when idle.  A task is a pair (frame F, index i): the
// candidate x = F.P[i] with Q-role = F.Q ∪ F.P[0..i-1] and P-role =
// F.P[i+1..] — exactly the sets Algorithm 1 holds when it pops x,
// because it retires x into Q unconditionally and never removes
// siblings from P.  So sibling tasks are independent and may run anywhere.
//
// Two task paths, chosen by |L| of the frame:
//  * list path (root frame, and frames with |L| > T): L' = L ∩ N(x) by warp
//    binary search; counts |N(v) ∩ L'| by REVERSE SCANNING
//    (P:510-528): for u ∈ L', for w ∈ N(u): cnt[w]++ (warp-flattened gather,
//    per-warp dense count table + touched list); roles by tag stamps.
//  * bit-row path (|L| <= T <= 128): every row of P ∪ Q is a bitmask over the
//    frame's L; L' = row(x); |N(v) ∩ L'| = popc(row(v) & row(x)); child rows
//    are column-compressed to L' coordinates.
// Maximality check: any Q-role v with |N(v) ∩ L'| = |L'| aborts
// the task.  Expansion: P-role c = |L'| → R', 0 < c < |L'| → P'.
// Children order P' by ascending (|N(v) ∩ L'|, r(v)) (iMBE).
// Two decision-preserving reductions: Q' rows are reduced to
// their antichain of maximal masks (R1), and among P-role siblings only an
// identical row can be a superset (R2), checked inside the equal-key block.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bits.cuh"
#include "mbe_internal.h"

#define FULLMASK 0xffffffffu
// Two instantiations of this file: the plain search (MBE_INSTR = 0, what runs in benchmarks) has
// every instrumentation path compiled out, keeping the hot code compact for the instruction cache;
// search_instr.cu includes it with MBE_INSTR = 1 for MBE_STATS, per-root counters and listings.
#ifndef MBE_INSTR
#define MBE_INSTR 0
#endif
#if MBE_INSTR
#define MBE_STATS_ON ((p.flags & F_STATS) != 0)
#define MBE_PER_ROOT (p.per_root)
#define MBE_CAP_RECORDS (p.cap_records)
#define MBE_EXPORT(name) name##_instr
#else
#define MBE_STATS_ON (false)
#define MBE_PER_ROOT ((unsigned long long*)nullptr)
#define MBE_CAP_RECORDS 0ull
#define MBE_EXPORT(name) name
#endif
#ifndef MBE_NARROW_TEMPLATES
#define MBE_NARROW_TEMPLATES 0  // bit mask: 2 / 4 = separate register-resident 2- / 4-word task bodies (0: only 1-word; smaller code, C5 -2 %)
#endif
#ifndef MBE_SCAN_MLP
#define MBE_SCAN_MLP 2  // reverse-scan visits in flight per lane (2 beat 1, 3, 4, 8 at the final build: C5 -3 %, C4 -6 %)
#endif
#ifndef MBE_BACKOFF_MIN
#define MBE_BACKOFF_MIN 64  // ns: first idle back-off after a failed steal attempt
#endif
#ifndef MBE_BACKOFF_MAX
#define MBE_BACKOFF_MAX 32768  // ns: cap of an idle warp's exponential back-off between steal attempts
#endif
#ifndef MBE_COMPRESS_ROWS
#define MBE_COMPRESS_ROWS 1  // wide column compression: rows per lane in flight (1 with a 2-way word unroll was best; 2 and 4 slower)
#endif
#ifndef MBE_COMPRESS_UNROLL
#define MBE_COMPRESS_UNROLL 1  // word-loop unroll of the wide column compression (1 beat 2 and 4: C5 -3 %, C4 -4 %)
#endif
constexpr int kCompressUnroll = MBE_COMPRESS_UNROLL;
#ifndef MBE_CLS_MLP
#define MBE_CLS_MLP 5  // touched-vertex slots in flight per lane during classification (r1: 2 -> 4, C5 80 -> 68 ms; r2 at 6 CTAs/SM: 5 beat 4 and 6, C4 -4.5 %, C3 -5 %, C5 -1.4 %)
#endif
#ifndef MBE_DEBUG_DELAYS
#define MBE_DEBUG_DELAYS 0  // 1: random __nanosleep at the claim / steal / publish / pop points (race stress builds)
#endif
#define KIND_LIST 0u
#define KIND_BITMAP 1u
#define HDR_UNCHECKED (1u << 16)  // frame header flag: Step 3 not yet run for its tasks (each task runs it)
#define TAG_R 0xffffffffu

namespace {

#ifndef SM_PROW_WORDS
#define SM_PROW_WORDS 128
#endif
#ifndef SM_QROW_WORDS
#define SM_QROW_WORDS 192
#endif
#define SM_RBUF 128
#ifndef FC_WORDS
#define FC_WORDS 256  // shared-memory copy of the warp's top frame (owner reads only)
#endif
#ifndef MBE_ACC_SMEM
#define MBE_ACC_SMEM 1  // lane-0 result accumulators in shared memory (frees registers: fewer spills on the task path)
#endif
#if MBE_ACC_SMEM
#define WACC(f) (w.sm->a_##f)
#else
#define WACC(f) (w.f)
#endif
struct __align__(16) WarpSmem {  // every array below starts at a 16-byte aligned offset
  union {                               // never live at the same time:
    unsigned long long skey[MBE_SMEM_SORT];  //   small sorts, antichain staging / wide metadata
    unsigned int hist[256];                  //   radix-sort histogram (keys then live in HBM)
  };
  unsigned int sval[MBE_SMEM_SORT];
  unsigned int foff[MBE_MAXDEPTH];  // arena word offset of the frame at each depth
  unsigned int fnp[MBE_MAXDEPTH];   // its task limit (|P|, or the end of a stolen range)
  unsigned int ffirst[MBE_MAXDEPTH];  // first task of its range (0 unless a thief's copy)
  unsigned int pend[MBE_MAXDEPTH];  // prefetched claim result (PEND_NONE = none)
  unsigned int pendk[MBE_MAXDEPTH]; // size of the prefetched claim
  unsigned int bcur[MBE_MAXDEPTH];  // owner's claimed batch [bcur, bend) at each depth
  unsigned int bend[MBE_MAXDEPTH];
  unsigned long long ph[16];        // MBE_STATS phase cycles (lane 0), see include/mbe.h
  unsigned int fcache[FC_WORDS];     // copy of the frame at depth fc_depth (16-B aligned)
  unsigned int fsz[MBE_MAXDEPTH];    // frame size in words per depth
  unsigned int lx[MBE_WMAX];         // row(x) of a wide (8/16-word) bit-row task
  int fc_depth;                      // depth held in fcache, -1 = none
  int pad_[3];
  unsigned long long wd_seen, wd_since;  // no-progress watchdog state (lane 0)
  union __align__(16) {
    unsigned short posv[32 * MBE_WMAX];  // wide tasks: column positions of row(x)'s set bits
    struct {                             // narrow tasks with small candidate bounds:
      unsigned int prow[SM_PROW_WORDS];  //   compressed P' candidate rows
      unsigned int qrow[SM_QROW_WORDS];  //   compressed Q' candidate rows
    };
  };
  unsigned int lbuf[128];            // L' ids
  unsigned int rbuf[SM_RBUF];        // expanded R' vertices
#if MBE_ACC_SMEM
  // lane-0 result accumulators (MBE_ACC_SMEM)
  unsigned long long a_count, a_hash, a_tasks, a_pruned, a_steals, a_list_tasks, a_bitmap_tasks, a_frames;
  unsigned long long a_ab_list, a_ab_bit, a_ab_write;
  unsigned int a_max_depth, a_pad;
#endif
};
#define PEND_NONE 0xffffffffu
#define SM_KEPT_WORDS (MBE_SMEM_SORT * 2)  // antichain kept list staged in skey's storage

struct Warp {
  int lane;
  uint32_t gw;
  // per-warp workspace base: the buffers are WB(slot), WB(touched), ... = base + the launch's offsets
  // (kernel-parameter constants), so no pointer per buffer stays live across the task code
  uint8_t* base;
  Desc* desc;
  uint32_t top;
  uint32_t atop;  // arena word offset of the next frame (Desc.off is 32-bit)
  uint32_t stamp;
  WarpSmem* sm;
  uint32_t cur_root;
  bool failed;
#if !MBE_ACC_SMEM
  // lane-0 accumulators
  unsigned long long count, hash, tasks, pruned, steals, list_tasks, bitmap_tasks, frames;
  unsigned long long ab_list, ab_bit, ab_write;  // MBE_STATS algorithmic bytes: list tasks, bit-row tasks, frame writes
  uint32_t max_depth;
#endif
};

// Per-warp buffers (api.cu ws_layout): slot [nU][MBE_SLOT_WORDS] (count, touched index + 1, tag lo, tag hi,
// bit-row words 0-3: one 32-B sector per vertex), and candidate-indexed: crow (bit-row words 4-15 of wide
// rows, in touched order), touched, lbuf, rbuf, skey, sval, pbuf, qbuf, plus the frame arena.
#define WB_T_slot uint32_t
#define WB_T_crow uint32_t
#define WB_T_touched uint32_t
#define WB_T_lbuf uint32_t
#define WB_T_rbuf uint32_t
#define WB_T_skey unsigned long long
#define WB_T_sval uint32_t
#define WB_T_pbuf uint32_t
#define WB_T_qbuf uint32_t
#define WB_T_arena uint32_t
#define WB(f) (reinterpret_cast<WB_T_##f*>(w.base + p.o_##f))

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}

__device__ __forceinline__ uint32_t ld_volatile(const unsigned int* p) { return *(volatile const unsigned int*)p; }
__device__ __forceinline__ unsigned long long ld_volatile64(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Race-stress builds (MBE_DEBUG_DELAYS=1, scripts/stress_delays.py): a random pause of up to ~4 us at
// one in four visits of every synchronisation point of the lock-free protocol.
__device__ __forceinline__ void dbg_delay(uint32_t salt) {
#if MBE_DEBUG_DELAYS
  uint32_t r = (uint32_t)clock64() * 0x9E3779B1u ^ salt * 0x85EBCA6Bu ^ (blockIdx.x << 7) ^ threadIdx.x;
  r ^= r >> 15;
  r *= 0x2C1B3C6Du;
  r ^= r >> 12;
  if ((r & 3u) == 0u) __nanosleep((r >> 8) & 4095u);
#else
  (void)salt;
#endif
}

// MBE_STATS sub-phase accounting: add the cycles since `t` to phase k and restart `t`.
#define MBE_PHASE(k, t)                                              \
  do {                                                               \
    if (MBE_STATS_ON && w.lane == 0) {                        \
      unsigned long long now_ = (unsigned long long)clock64();       \
      w.sm->ph[k] += now_ - (t);                                     \
      atomicMax(&p.gl->max_phase[k], now_ - (t));                    \
      (t) = now_;                                                    \
    }                                                                \
  } while (0)

__device__ __forceinline__ void set_error(const SearchParams& p, unsigned int code, unsigned long long info) {
  if (atomicCAS(&p.gl->error, 0u, code) == 0u) p.gl->err_info = info;
}

// ------------------------------------------------------------------ rows
template <int W>
struct Row {
  uint32_t w[W];
};

template <int W>
__device__ __forceinline__ Row<W> load_row(const uint32_t* p) {
  Row<W> r;
  if constexpr (W == 1) {
    r.w[0] = *p;
  } else if constexpr (W == 2) {
    uint2 v = *reinterpret_cast<const uint2*>(p);
    r.w[0] = v.x;
    r.w[1] = v.y;
  } else {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    r.w[0] = v.x;
    r.w[1] = v.y;
    r.w[2] = v.z;
    r.w[3] = v.w;
  }
  return r;
}

template <int W>
__device__ __forceinline__ void store_row(uint32_t* p, const Row<W>& r) {
  if constexpr (W == 1) {
    *p = r.w[0];
  } else if constexpr (W == 2) {
    *reinterpret_cast<uint2*>(p) = make_uint2(r.w[0], r.w[1]);
  } else {
    *reinterpret_cast<uint4*>(p) = make_uint4(r.w[0], r.w[1], r.w[2], r.w[3]);
  }
}

template <int W>
__device__ __forceinline__ Row<W> zero_row() {
  Row<W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.w[k] = 0;
  return r;
}

template <int W>
__device__ __forceinline__ Row<W> shfl_row(const Row<W>& r, int src) {
  Row<W> o;
#pragma unroll
  for (int k = 0; k < W; ++k) o.w[k] = __shfl_sync(FULLMASK, r.w[k], src);
  return o;
}

template <int W>
__device__ __forceinline__ bool row_subset(const Row<W>& a, const Row<W>& b) {  // a ⊆ b
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) x |= a.w[k] & ~b.w[k];
  return x == 0;
}

template <int W>
__device__ __forceinline__ bool row_eq(const Row<W>& a, const Row<W>& b) {
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) x |= a.w[k] ^ b.w[k];
  return x == 0;
}

template <int W>
__device__ __forceinline__ uint32_t row_popc_and(const Row<W>& a, const Row<W>& b) {
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) c += __popc(a.w[k] & b.w[k]);
  return c;
}

template <int W>
__device__ __forceinline__ bool row_any_and(const Row<W>& a, const Row<W>& b) {
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) x |= a.w[k] & b.w[k];
  return x != 0;
}

// ------------------------------------------------------------------ sorting
// Ascending sort of n (key, val) pairs in place (keys unique: (count << 32) | id).
#ifndef MBE_AC_ROLL
#define MBE_AC_ROLL 1
#endif
// n <= 32 pairs: rank sort (keys are unique), one rolled loop — a tiny instruction footprint
// for the most frequent sort of the search (the P' candidates of a bit-row child).
__device__ __noinline__ void sort_regs32(unsigned long long* key, uint32_t* val, uint32_t n, int lane) {
  const bool mine = lane < (int)n;
  const unsigned long long k = mine ? key[lane] : ~0ull;
  const uint32_t v = mine ? val[lane] : 0u;
  uint32_t rank = 0;
#pragma unroll 1
  for (uint32_t s = 0; s < n; ++s) rank += __shfl_sync(FULLMASK, k, s) < k ? 1u : 0u;
  __syncwarp();
  if (mine) {
    key[rank] = k;
    val[rank] = v;
  }
  __syncwarp();
}

__device__ __noinline__ void sort_smem(unsigned long long* key, uint32_t* val, uint32_t n, WarpSmem* sm, int lane) {
  uint32_t N = 64;
  while (N < n) N <<= 1;
  for (uint32_t t = lane; t < N; t += 32) {
    sm->skey[t] = t < n ? key[t] : ~0ull;
    sm->sval[t] = t < n ? val[t] : 0u;
  }
  __syncwarp();
  for (uint32_t size = 2; size <= N; size <<= 1) {
    for (uint32_t j = size >> 1; j > 0; j >>= 1) {
      for (uint32_t t = lane; t < N / 2; t += 32) {
        uint32_t i = (t / j) * 2 * j + (t % j);
        uint32_t l = i + j;
        bool up = (i & size) == 0;
        unsigned long long a = sm->skey[i], b = sm->skey[l];
        if ((a > b) == up) {
          sm->skey[i] = b;
          sm->skey[l] = a;
          uint32_t va = sm->sval[i];
          sm->sval[i] = sm->sval[l];
          sm->sval[l] = va;
        }
      }
      __syncwarp();
    }
  }
  for (uint32_t t = lane; t < n; t += 32) {
    key[t] = sm->skey[t];
    val[t] = sm->sval[t];
  }
  __syncwarp();
}

// Stable LSD radix sort with 8-bit digits over the significant bits of
// key = (count << 32) | id.  Ping-pong between (key,val) and (key2,val2).
__device__ __noinline__ void sort_radix(unsigned long long* key, uint32_t* val, unsigned long long* key2, uint32_t* val2,
                           uint32_t n, uint32_t id_bits, uint32_t cnt_bits, WarpSmem* sm, int lane) {
  unsigned long long* src_k = key;
  uint32_t* src_v = val;
  unsigned long long* dst_k = key2;
  uint32_t* dst_v = val2;
  uint32_t shifts[8];
  int np = 0;
  for (uint32_t s = 0; s < id_bits; s += 8) shifts[np++] = s;
  for (uint32_t s = 0; s < cnt_bits; s += 8) shifts[np++] = 32 + s;
#pragma unroll 1
  for (int pass = 0; pass < np; ++pass) {
    uint32_t sh = shifts[pass];
    for (int b = lane; b < 256; b += 32) sm->hist[b] = 0;
    __syncwarp();
#pragma unroll 1
    for (uint32_t t = lane; t < n; t += 32) atomicAdd(&sm->hist[(src_k[t] >> sh) & 255u], 1u);
    __syncwarp();
    // exclusive scan of 256 buckets: lane owns 8 consecutive buckets
    uint32_t loc[8];
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      loc[q] = sm->hist[lane * 8 + q];
      s += loc[q];
    }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t run = incl - s;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      sm->hist[lane * 8 + q] = run;
      run += loc[q];
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t base = 0; base < n; base += 32) {
      uint32_t t = base + lane;
      bool valid = t < n;
      unsigned long long k = valid ? src_k[t] : 0ull;
      uint32_t v = valid ? src_v[t] : 0u;
      uint32_t d = valid ? (uint32_t)((k >> sh) & 255u) : 256u + lane;
      uint32_t peers = __match_any_sync(FULLMASK, d);
      uint32_t rank = __popc(peers & lanemask_lt());
      uint32_t pos = valid ? sm->hist[d] + rank : 0u;
      __syncwarp();
      if (valid && rank == (uint32_t)__popc(peers) - 1u) sm->hist[d] += (uint32_t)__popc(peers);
      if (valid) {
        dst_k[pos] = k;
        dst_v[pos] = v;
      }
      __syncwarp();
    }
    unsigned long long* tk = src_k;
    src_k = dst_k;
    dst_k = tk;
    uint32_t* tv = src_v;
    src_v = dst_v;
    dst_v = tv;
  }
  if (src_k != key) {
#pragma unroll 1
    for (uint32_t t = lane; t < n; t += 32) {
      key[t] = src_k[t];
      val[t] = src_v[t];
    }
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t bit_length(uint32_t x) { return x ? 32u - __clz(x) : 0u; }

// Sort keys of child candidates (mbe_config.order): ascending (c, r) is the paper's iMBE order
// (P:491-493); the input (r) and descending (-c, r) orders are the ablation.
// c = |N(v) ∩ L'| < maxc, v = r(v) (internal id = position in the root order).
__device__ __forceinline__ unsigned long long order_key(uint32_t order, uint32_t c, uint32_t v, uint32_t maxc) {
  if (order == 1u) return ((unsigned long long)v << 32) | c;
  return ((unsigned long long)(order == 2u ? maxc - c : c) << 32) | v;
}
__device__ __forceinline__ uint32_t key_id(uint32_t order, unsigned long long k) {
  return order == 1u ? (uint32_t)(k >> 32) : (uint32_t)k;
}
__device__ __forceinline__ uint32_t key_count(uint32_t order, unsigned long long k, uint32_t maxc) {
  return order == 1u ? (uint32_t)k : (order == 2u ? maxc - (uint32_t)(k >> 32) : (uint32_t)(k >> 32));
}

__device__ __noinline__ void sort_pairs_small(unsigned long long* key, uint32_t* val, uint32_t n, WarpSmem* sm, int lane) {
  if (n <= 1) return;
  if (n <= 32) sort_regs32(key, val, n, lane);
  else sort_smem(key, val, n, sm, lane);
}

__device__ void warp_sort_pairs(Warp& w, const SearchParams& p, uint32_t n, uint32_t max_count) {
  if (n <= 1) return;
  if (n <= 32) {
    sort_regs32(WB(skey), WB(sval), n, w.lane);
  } else if (n <= MBE_SMEM_SORT) {
    sort_smem(WB(skey), WB(sval), n, w.sm, w.lane);
  } else {
    // second buffers live right after the first ones (same per-warp region, sized nU)
    unsigned long long* key2 = WB(skey) + p.skey2_off;
    uint32_t* val2 = WB(sval) + p.skey2_off;
    const uint32_t ib = bit_length(p.g.nU), cb = bit_length(max_count);
    if (p.order == 1u) sort_radix(WB(skey), WB(sval), key2, val2, n, cb, ib, w.sm, w.lane);
    else sort_radix(WB(skey), WB(sval), key2, val2, n, ib, cb, w.sm, w.lane);
  }
}

// ------------------------------------------------------------------ antichain (R1)
// Reduce n candidate rows (src, W words each) to the set of distinct maximal
// rows under inclusion, written to dst.  Decision-preserving: a later check
// "∃q: L'' ⊆ N(q)" holds for a dominated row only if it holds for its
// dominator.  With keep_all, rows are copied unchanged.
template <int W>
__device__ __noinline__ uint32_t antichain(const uint32_t* src, uint32_t n, uint32_t* dst, bool keep_all, int lane,
                                           bool sorted_desc = false) {
  if (keep_all) {
    for (uint32_t t = lane; t < n; t += 32) store_row<W>(dst + (size_t)t * W, load_row<W>(src + (size_t)t * W));
    __syncwarp();
    return n;
  }
  uint32_t K = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    bool valid = base + lane < n;
    Row<W> r = valid ? load_row<W>(src + (size_t)(base + lane) * W) : zero_row<W>();
    bool dom = !valid;
    // kept rows in blocks of 32: one coalesced load per lane, then 32 register shuffles
    for (uint32_t kb = 0; kb < K; kb += 32) {
      const bool kval = kb + lane < K;
      const Row<W> kr = kval ? load_row<W>(dst + (size_t)(kb + lane) * W) : zero_row<W>();
      const uint32_t nk = min(32u, K - kb);
#if MBE_AC_ROLL
#pragma unroll 1
#endif
      for (uint32_t m = 0; m < nk; ++m) {
        const Row<W> km = shfl_row<W>(kr, (int)m);
        if (row_subset<W>(r, km)) dom = true;
      }
    }
    // intra-chunk dominance: only the valid candidates of this chunk (usually a handful)
    const int nv = (int)min(32u, n - base);
#if MBE_AC_ROLL
#pragma unroll 1
#endif
    for (int m = 0; m < nv; ++m) {
      Row<W> mr = shfl_row<W>(r, m);
      if (m != lane && row_subset<W>(r, mr) && (!row_eq<W>(r, mr) || m < lane)) dom = true;
    }
    bool surv = valid && !dom;
    uint32_t bs = __ballot_sync(FULLMASK, surv);
    if (bs && sorted_desc) {
      // candidates arrive by descending popcount: a survivor cannot strictly contain a kept row
      if (surv) store_row<W>(dst + (size_t)(K + __popc(bs & lanemask_lt())) * W, r);
      K += __popc(bs);
      __syncwarp();
    } else if (bs) {
      uint32_t newK = 0;
      for (uint32_t kb = 0; kb < K; kb += 32) {
        bool kval = kb + lane < K;
        Row<W> kr = kval ? load_row<W>(dst + (size_t)(kb + lane) * W) : zero_row<W>();
        bool kdom = false;
        uint32_t rem = bs;
        while (rem) {
          int m = __ffs(rem) - 1;
          rem &= rem - 1;
          Row<W> sr = shfl_row<W>(r, m);
          if (kval && row_subset<W>(kr, sr)) kdom = true;
        }
        bool keep = kval && !kdom;
        uint32_t bk = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) store_row<W>(dst + (size_t)(newK + __popc(bk & lanemask_lt())) * W, kr);
        newK += __popc(bk);
        __syncwarp();
      }
      K = newK;
      if (surv) store_row<W>(dst + (size_t)(K + __popc(bs & lanemask_lt())) * W, r);
      K += __popc(bs);
      __syncwarp();
    }
  }
  return K;
}

// Exact-duplicate removal before the antichain for large candidate sets: sort
// the rows by (popcount descending, 32-bit row hash) with the warp radix sort,
// then keep a row unless it equals its predecessor.  Output rows are in
// descending popcount order.  (Equal rows get equal keys; distinct rows that
// collide on the hash are compared word by word, so the result is exact.)
__device__ __noinline__ uint32_t dedup_sort_rows(const uint32_t* src, uint32_t n, uint32_t W, uint32_t* dst,
                                                 unsigned long long* key, uint32_t* val, unsigned long long* key2,
                                                 uint32_t* val2, WarpSmem* sm, int lane) {
  for (uint32_t t = lane; t < n; t += 32) {
    const uint32_t* r = src + (size_t)t * W;
    uint32_t pc = 0, h = 0x9E3779B9u;
    for (uint32_t q = 0; q < W; ++q) {
      const uint32_t a = r[q];
      pc += __popc(a);
      h = (h ^ a) * 0x01000193u;
      h ^= h >> 15;
    }
    key[t] = ((unsigned long long)(W * 32u - pc) << 32) | (h & 0xffffffu);
    val[t] = t;
  }
  __syncwarp();
  sort_radix(key, val, key2, val2, n, 24, bit_length(W * 32u), sm, lane);
  uint32_t m = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t t = base + lane;
    bool keep = false;
    if (t < n) {
      keep = true;
      if (t > 0 && key[t] == key[t - 1]) {
        const uint32_t* a = src + (size_t)val[t] * W;
        const uint32_t* b = src + (size_t)val[t - 1] * W;
        uint32_t x = 0;
        for (uint32_t q = 0; q < W; ++q) x |= a[q] ^ b[q];
        keep = x != 0u;
      }
    }
    const uint32_t bk = __ballot_sync(FULLMASK, keep);
    if (keep) {
      const uint32_t* a = src + (size_t)val[t] * W;
      uint32_t* o = dst + (size_t)(m + __popc(bk & lanemask_lt())) * W;
      for (uint32_t q = 0; q < W; ++q) o[q] = a[q];
    }
    m += __popc(bk);
  }
  __syncwarp();
  return m;
}

// Exact duplicate removal by hashing (O(n), one table round trip per row).
// table: 2^cap_log2 >= 2n u64 entries of scratch (cleared here first).
// Entry = (hash32 << 32) | (row index + 1), claimed by CAS; on a hash match the
// rows are compared word by word, so the result is exact.  Output rows keep
// first-occurrence order; returns the number of distinct rows.
__device__ __noinline__ uint32_t dedup_hash_rows(const uint32_t* src, uint32_t n, uint32_t W, uint32_t* dst,
                                                 unsigned long long* table, uint32_t cap_log2, int lane) {
  const uint32_t cap = 1u << cap_log2, mask = cap - 1;
  for (uint32_t k = lane; k < cap; k += 32) table[k] = 0ull;
  __syncwarp();
  uint32_t m = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t t = base + lane;
    bool keep = false;
    if (t < n) {
      const uint32_t* r = src + (size_t)t * W;
      uint32_t h = 0x9E3779B9u;
      for (uint32_t q = 0; q < W; ++q) {
        h = (h ^ r[q]) * 0x01000193u;
        h ^= h >> 15;
      }
      h = h * 0x85EBCA6Bu;
      h ^= h >> 13;
      // lanes of this step holding the same row: only the lowest one probes the table (equal rows
      // in one warp step would otherwise serialise their CAS on one entry)
      const uint32_t peers = __match_any_sync(__activemask(), h);
      const int lead = __ffs(peers) - 1;
      if (lead != lane) {
        const uint32_t* o = src + (size_t)(base + lead) * W;
        bool eq = true;
        for (uint32_t q = 0; q < W && eq; ++q) eq = o[q] == r[q];
        if (eq) goto decided;  // duplicate of the leader's row (the leader keeps or drops it)
      }
      {
      const unsigned long long mine = ((unsigned long long)h << 32) | (t + 1);
      uint32_t slot = h & mask;
      for (;;) {
        const unsigned long long old = atomicCAS(&table[slot], 0ull, mine);
        if (old == 0ull) {
          keep = true;
          break;
        }
        if ((uint32_t)(old >> 32) == h) {
          const uint32_t* o = src + (size_t)((uint32_t)old - 1) * W;
          bool eq = true;
          for (uint32_t q = 0; q < W && eq; ++q) eq = o[q] == r[q];
          if (eq) break;  // duplicate of an earlier-inserted row
        }
        slot = (slot + 1) & mask;
      }
      }
    decided:;
    }
    const uint32_t bk = __ballot_sync(FULLMASK, keep);
    if (keep) {
      const uint32_t* r = src + (size_t)t * W;
      uint32_t* o = dst + (size_t)(m + __popc(bk & lanemask_lt())) * W;
      for (uint32_t q = 0; q < W; ++q) o[q] = r[q];
    }
    m += __popc(bk);
  }
  __syncwarp();
  return m;
}

// R1 pre-filter (exact, O(n · popcount)): champ[c] = the row of largest popcount (lowest index on ties)
// having column c.  A row contained in the champion of one of its columns is dropped: a strictly contained
// row is dominated, an equal row is a later copy of the champion.  Every distinct maximal row keeps a copy,
// so the antichain of the survivors is the antichain of all n rows; most rows of a hub's Q' (a handful of
// columns each) go here instead of through the O(n · K) pass.  W <= 8 words, k <= 32 W columns, n < 2^22.
#ifndef MBE_CHAMP_MIN
#define MBE_CHAMP_MIN 128u  // list-path Q' candidate sets above this go through the champion filter (0: off)
#endif
#define CHAMP_IDX 0x3FFFFFu
__device__ __noinline__ uint32_t champion_filter(const uint32_t* src, uint32_t n, uint32_t W, uint32_t k, uint32_t* dst,
                                                 uint32_t* champ, int lane) {
  for (uint32_t c = lane; c < k; c += 32) champ[c] = 0u;
  __syncwarp();
  for (uint32_t t = lane; t < n; t += 32) {
    const uint32_t* r = src + (size_t)t * W;
    uint32_t pc = 0;
    for (uint32_t q = 0; q < W; ++q) pc += __popc(r[q]);
    const uint32_t key = (pc << 22) | (CHAMP_IDX - t);
    for (uint32_t q = 0; q < W; ++q)
      for (uint32_t m = r[q]; m; m &= m - 1u) atomicMax(&champ[32 * q + __ffs(m) - 1], key);
  }
  __syncwarp();
  uint32_t out = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t t = base + lane;
    bool keep = t < n;
    const uint32_t* r = src + (size_t)(keep ? t : 0u) * W;
    for (uint32_t q = 0, seen = 0; q < W && keep && seen < 8; ++q)
      for (uint32_t m = r[q]; m && keep && seen < 8; m &= m - 1u, ++seen) {
        const uint32_t j = CHAMP_IDX - (champ[32 * q + __ffs(m) - 1] & CHAMP_IDX);
        if (j == t) continue;
        const uint32_t* o = src + (size_t)j * W;
        uint32_t x = 0;
        for (uint32_t qq = 0; qq < W; ++qq) x |= r[qq] & ~o[qq];
        if (x == 0u) keep = false;
      }
    const uint32_t bk = __ballot_sync(FULLMASK, keep);
    if (keep) {
      uint32_t* d = dst + (size_t)(out + __popc(bk & lanemask_lt())) * W;
      for (uint32_t q = 0; q < W; ++q) d[q] = r[q];
    }
    out += __popc(bk);
  }
  __syncwarp();
  return out;
}

// Same reduction for wide rows (8 or 16 words), word-sliced: rows are streamed from
// memory (L1) instead of held in registers.
#ifndef MBE_VEC_SUBSET
#define MBE_VEC_SUBSET 0
#endif
#ifndef MBE_META54
#define MBE_META54 1
#endif
#if MBE_VEC_SUBSET
// Rows are 16-byte aligned and W is 8 or 16: all words are read with vector loads in flight at once.
__device__ __forceinline__ bool wide_subset(const uint32_t* a, const uint32_t* b, uint32_t W) {  // a ⊆ b
  uint32_t x = 0;
#pragma unroll
  for (uint32_t q = 0; q < MBE_WMAX; q += 4)
    if (q < W) {
      const uint4 u = *reinterpret_cast<const uint4*>(a + q), v = *reinterpret_cast<const uint4*>(b + q);
      x |= (u.x & ~v.x) | (u.y & ~v.y) | (u.z & ~v.z) | (u.w & ~v.w);
    }
  return x == 0u;
}
__device__ __forceinline__ bool wide_eq(const uint32_t* a, const uint32_t* b, uint32_t W) {
  uint32_t x = 0;
#pragma unroll
  for (uint32_t q = 0; q < MBE_WMAX; q += 4)
    if (q < W) {
      const uint4 u = *reinterpret_cast<const uint4*>(a + q), v = *reinterpret_cast<const uint4*>(b + q);
      x |= (u.x ^ v.x) | (u.y ^ v.y) | (u.z ^ v.z) | (u.w ^ v.w);
    }
  return x == 0u;
}
#else
__device__ __forceinline__ bool wide_subset(const uint32_t* a, const uint32_t* b, uint32_t W) {  // a ⊆ b
  for (uint32_t q = 0; q < W; ++q)  // early exit: most non-subset pairs fail within a word or two
    if (a[q] & ~b[q]) return false;
  return true;
}
__device__ __forceinline__ bool wide_eq(const uint32_t* a, const uint32_t* b, uint32_t W) {
  for (uint32_t q = 0; q < W; ++q)
    if (a[q] != b[q]) return false;
  return true;
}
#endif

// Necessary-condition filters for wide rows: a ⊆ b requires popc(a) <= popc(b) and
// fold(a) ⊆ fold(b); a == b requires equal metadata.
#ifndef MBE_META_ROLL
#define MBE_META_ROLL 0  // 1: the wide-row metadata loop is not unrolled
#endif
#if MBE_META54
// fold = OR of the row's 64-bit halves (54 buckets kept); meta = (popc << 54) | fold
#define MBE_META_SHIFT 54
#define MBE_META_FOLD ((1ull << 54) - 1ull)
__device__ __forceinline__ unsigned long long wide_meta(const uint32_t* r, uint32_t W) {
  uint32_t pc = 0;
  unsigned long long f = 0;
#if MBE_META_ROLL
#pragma unroll 1
  for (uint32_t q = 0; q < W; q += 4) {
#else
#pragma unroll
  for (uint32_t q = 0; q < MBE_WMAX; q += 4)
    if (q < W) {
#endif
      const uint4 u = *reinterpret_cast<const uint4*>(r + q);
      pc += __popc(u.x) + __popc(u.y) + __popc(u.z) + __popc(u.w);
      f |= ((unsigned long long)u.y << 32 | u.x) | ((unsigned long long)u.w << 32 | u.z);
    }
  return ((unsigned long long)pc << 54) | (f & MBE_META_FOLD);
}
#else
// fold = OR of the row's words; meta = (popc << 32) | fold
#define MBE_META_SHIFT 32
#define MBE_META_FOLD 0xffffffffull
__device__ __forceinline__ unsigned long long wide_meta(const uint32_t* r, uint32_t W) {
  uint32_t pc = 0, f = 0;
  for (uint32_t q = 0; q < W; ++q) {
    const uint32_t a = r[q];
    pc += __popc(a);
    f |= a;
  }
  return ((unsigned long long)pc << 32) | f;
}
#endif
__device__ __forceinline__ bool meta_may_subset(unsigned long long a, unsigned long long b) {
  return (a >> MBE_META_SHIFT) <= (b >> MBE_META_SHIFT) && (a & ~b & MBE_META_FOLD) == 0ull;
}

__device__ __noinline__ uint32_t antichain_wide(const uint32_t* src, uint32_t n, uint32_t* dst, uint32_t W, bool keep_all,
                                   int lane, unsigned long long* kmeta /* smem [MBE_SMEM_SORT] */,
                                   unsigned long long* kmeta_g /* global spill for kept rows >= MBE_SMEM_SORT, or null */) {
  if (keep_all) {
    for (uint32_t t = lane; t < n * W; t += 32) dst[t] = src[t];
    __syncwarp();
    return n;
  }
  uint32_t K = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t t = base + lane;
    const bool valid = t < n;
    const uint32_t* r = src + (size_t)(valid ? t : 0) * W;
    const unsigned long long mr = valid ? wide_meta(r, W) : 0ull;
    bool dom = !valid;
    // kept rows in blocks of 32: lane l fetches the (popc, fold) of kept row kb+l, then the
    // block is broadcast by shuffles; only pairs passing the filter stream their words
    for (uint32_t kb = 0; kb < K; kb += 32) {
      const uint32_t kk = kb + lane;
      const unsigned long long mkl =
          kk < K ? (kk < MBE_SMEM_SORT ? kmeta[kk] : (kmeta_g ? kmeta_g[kk] : wide_meta(dst + (size_t)kk * W, W)))
                 : ~0ull;
      const uint32_t nk = min(32u, K - kb);
#if MBE_AC_ROLL
#pragma unroll 1
#endif
      for (uint32_t m = 0; m < nk; ++m) {
        const unsigned long long mk = __shfl_sync(FULLMASK, mkl, (int)m);
        if (!dom && meta_may_subset(mr, mk) && wide_subset(r, dst + (size_t)(kb + m) * W, W)) dom = true;
      }
    }
    const int nv = (int)min(32u, n - base);
#if MBE_AC_ROLL
#pragma unroll 1
#endif
    for (int m = 0; m < nv; ++m) {
      const unsigned long long mm = __shfl_sync(FULLMASK, mr, m);
      if (!dom && m != lane && meta_may_subset(mr, mm)) {
        const uint32_t* o = src + (size_t)(base + m) * W;
        if (wide_subset(r, o, W) && (m < lane || !wide_eq(r, o, W))) dom = true;
      }
    }
    const bool surv = valid && !dom;
    const uint32_t bs = __ballot_sync(FULLMASK, surv);
    if (bs) {
      uint32_t newK = 0;
      for (uint32_t kb = 0; kb < K; kb += 32) {
        const bool kval = kb + lane < K;
        const uint32_t kk = kval ? kb + lane : 0u;
        const uint32_t* kr = dst + (size_t)kk * W;
        const unsigned long long mk =
            kval ? (kk < MBE_SMEM_SORT ? kmeta[kk] : (kmeta_g ? kmeta_g[kk] : wide_meta(kr, W))) : 0ull;
        bool kdom = false;
        for (int m = 0; m < 32; ++m) {
          const unsigned long long ms = __shfl_sync(FULLMASK, mr, m);
          if (((bs >> m) & 1u) && kval && !kdom && meta_may_subset(mk, ms) &&
              wide_subset(kr, src + (size_t)(base + m) * W, W))
            kdom = true;
        }
        const bool keep = kval && !kdom;
        uint32_t row[MBE_WMAX];
        for (uint32_t q = 0; q < W; ++q) row[q] = keep ? kr[q] : 0u;
        const uint32_t bk = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) {
          const uint32_t ni = newK + __popc(bk & lanemask_lt());
          uint32_t* o = dst + (size_t)ni * W;
          for (uint32_t q = 0; q < W; ++q) o[q] = row[q];
          if (ni < MBE_SMEM_SORT) kmeta[ni] = mk;
          else if (kmeta_g) kmeta_g[ni] = mk;
        }
        newK += __popc(bk);
        __syncwarp();
      }
      K = newK;
      if (surv) {
        const uint32_t ni = K + __popc(bs & lanemask_lt());
        uint32_t* o = dst + (size_t)ni * W;
        for (uint32_t q = 0; q < W; ++q) o[q] = r[q];
        if (ni < MBE_SMEM_SORT) kmeta[ni] = mr;
        else if (kmeta_g) kmeta_g[ni] = mr;
      }
      K += __popc(bs);
      __syncwarp();
    }
  }
  return K;
}

// Rows reordered by descending popcount (counting sort; order inside a popcount is arbitrary).
// hist: shared memory with >= 32*W + 1 entries.
__device__ __noinline__ void popc_sort_rows_desc(const uint32_t* src, uint32_t n, uint32_t W, uint32_t* dst,
                                                 uint32_t* hist, int lane) {
  const uint32_t nb = 32 * W + 1;
  for (uint32_t b = lane; b < nb; b += 32) hist[b] = 0;
  __syncwarp();
  for (uint32_t t = lane; t < n; t += 32) {
    uint32_t pc = 0;
    for (uint32_t q = 0; q < W; ++q) pc += __popc(src[(size_t)t * W + q]);
    atomicAdd(&hist[32 * W - pc], 1u);
  }
  __syncwarp();
  if (lane == 0) {
    uint32_t run = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      const uint32_t c = hist[b];
      hist[b] = run;
      run += c;
    }
  }
  __syncwarp();
  for (uint32_t t = lane; t < n; t += 32) {
    uint32_t pc = 0;
    for (uint32_t q = 0; q < W; ++q) pc += __popc(src[(size_t)t * W + q]);
    const uint32_t pos = atomicAdd(&hist[32 * W - pc], 1u);
    for (uint32_t q = 0; q < W; ++q) dst[(size_t)pos * W + q] = src[(size_t)t * W + q];
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t antichain_w(uint32_t Wc, const uint32_t* src, uint32_t n, uint32_t* dst,
                                                bool keep_all, int lane, WarpSmem* sm,
                                                unsigned long long* kmeta_g = nullptr, bool sorted_desc = false) {
  if (Wc == 1) return antichain<1>(src, n, dst, keep_all, lane, sorted_desc);
  if (Wc == 2) return antichain<2>(src, n, dst, keep_all, lane, sorted_desc);
  if (Wc == 4) return antichain<4>(src, n, dst, keep_all, lane, sorted_desc);
  return antichain_wide(src, n, dst, Wc, keep_all, lane, sm->skey, kmeta_g);
}

// ------------------------------------------------------------------ misc
__device__ __forceinline__ bool bsearch_u32(const uint32_t* a, uint32_t n, uint32_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    uint32_t x = a[mid];
    if (x < v) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && a[lo] == v;
}

// out = A ∩ B (both sorted ascending), in ascending order; returns |out|.
__device__ __noinline__ uint32_t warp_intersect(const uint32_t* A, uint32_t nA, const uint32_t* B, uint32_t nB, uint32_t* out,
                                   int lane) {
  if (nA > nB) {
    const uint32_t* t = A;
    A = B;
    B = t;
    uint32_t tn = nA;
    nA = nB;
    nB = tn;
  }
  uint32_t c = 0;
  for (uint32_t base = 0; base < nA; base += 32) {
    bool valid = base + lane < nA;
    uint32_t v = valid ? A[base + lane] : 0u;
    bool f = valid && bsearch_u32(B, nB, v);
    uint32_t b = __ballot_sync(FULLMASK, f);
    if (f) out[c + __popc(b & lanemask_lt())] = v;
    c += __popc(b);
  }
  __syncwarp();
  return c;
}

__device__ __forceinline__ uint64_t align4(uint64_t x) { return (x + 3) & ~3ull; }

// Per-task accounting (tasks/pruned), lane 0.
__device__ __forceinline__ void account_task(Warp& w, const SearchParams& p, bool pruned) {
  if (w.lane == 0) {
    WACC(tasks)++;
    if (pruned) WACC(pruned)++;
    if (MBE_PER_ROOT) {
      atomicAdd(&MBE_PER_ROOT[(size_t)w.cur_root * 4 + 2], 1ull);
      if (pruned) atomicAdd(&MBE_PER_ROOT[(size_t)w.cur_root * 4 + 3], 1ull);
    }
  }
}

__device__ __forceinline__ void account_emit(Warp& w, const SearchParams& p, uint64_t sL, uint32_t nL, uint64_t sR,
                                             uint32_t nR) {
  if (w.lane == 0) {
    uint64_t h = mbe_biclique_hash(p.cand_side, sL, nL, sR, nR);
    WACC(count)++;
    WACC(hash) += h;
    if (MBE_PER_ROOT) {
      atomicAdd(&MBE_PER_ROOT[(size_t)w.cur_root * 4 + 0], 1ull);
      atomicAdd(&MBE_PER_ROOT[(size_t)w.cur_root * 4 + 1], (unsigned long long)h);
    }
  }
}

// Bounded listing: record (A, B) in original ids.  Lids: L' (V ids) sorted;
// R' = Rfr (frame R, U ranks) ∪ {x} ∪ rexp (U ranks).
__device__ __noinline__ void write_record(const int lane, const SearchParams& p, const uint32_t* Lids, uint32_t nL, const uint32_t* Rfr,
                             uint32_t nRf, uint32_t x, const uint32_t* rexp, uint32_t nRx) {
  uint32_t nR = nRf + 1 + nRx;
  unsigned long long rec = 0, ido = 0;
  if (lane == 0) {
    rec = atomicAdd(&p.gl->out_records, 1ull);
    ido = atomicAdd(&p.gl->out_ids, (unsigned long long)(nL + nR));
  }
  rec = __shfl_sync(FULLMASK, rec, 0);
  ido = __shfl_sync(FULLMASK, ido, 0);
  if (rec >= MBE_CAP_RECORDS) return;
  if (ido + nL + nR > p.cap_ids) {
    if (lane == 0) p.rec_off[rec] = ~0ull;  // record counted but its ids did not fit
    return;
  }
  uint32_t nA = p.cand_side == 1 ? nR : nL;
  uint32_t nB = p.cand_side == 1 ? nL : nR;
  uint32_t offR = p.cand_side == 1 ? 0u : nL;
  uint32_t offL = p.cand_side == 1 ? nR : 0u;
  unsigned int* ids = p.out_ids + ido;
  for (uint32_t t = lane; t < nL; t += 32) ids[offL + t] = Lids[t];
  for (uint32_t t = lane; t < nR; t += 32) {
    uint32_t r = t < nRf ? Rfr[t] : (t == nRf ? x : rexp[t - nRf - 1]);
    ids[offR + t] = p.g.origU[r];
  }
  if (lane == 0) {
    p.rec_off[rec] = ido;
    p.rec_n1[rec] = nA;
    p.rec_n2[rec] = nB;
  }
  __syncwarp();
}

// Reserve space for a child frame at the top of the arena; false on overflow.
__device__ __forceinline__ bool arena_reserve(Warp& w, const SearchParams& p, uint64_t words) {
  if (w.atop + words + 8 > p.arena_words || w.top + 1 >= MBE_MAXDEPTH) {
    if (w.lane == 0) set_error(p, w.top + 1 >= MBE_MAXDEPTH ? 2u : 1u, w.atop + words);
    w.failed = true;
    return false;
  }
  if (MBE_STATS_ON && w.lane == 0) atomicMax(&p.gl->max_arena_words, (unsigned long long)(w.atop + words));
  return true;
}

// Publish the frame just written at arena offset w.atop (size words) as depth w.top.
__device__ void publish_frame(Warp& w, const SearchParams& p, uint64_t size_words, uint32_t nP,
                              uint32_t first = 0u) {
  __syncwarp();
  if (w.lane == 0) {
    Desc* d = &w.desc[w.top];
    d->off = (unsigned int)w.atop;
    d->done = 0u;
    d->size = (unsigned int)size_words;
    d->first = first;
    w.sm->foff[w.top] = (unsigned int)w.atop;
    w.sm->fnp[w.top] = nP;
    w.sm->ffirst[w.top] = first;
    w.sm->pend[w.top] = PEND_NONE;
    w.sm->bcur[w.top] = 0u;
    w.sm->bend[w.top] = 0u;
    w.sm->fsz[w.top] = (unsigned int)size_words;
    if (w.sm->fc_depth == (int)w.top) w.sm->fc_depth = -1;
    __threadfence();
    dbg_delay(1);
    atomicExch(&d->claim, (((unsigned long long)nP) << 32) | first);
    p.tops[w.gw] = w.top + 1;
    if (nP - first >= 2 && !(p.flags & F_NO_STEAL)) atomicOr(&p.hint[w.gw >> 5], 1u << (w.gw & 31));
    WACC(frames)++;
  }
  w.atop = align4(w.atop + size_words);
  w.top += 1;
  if (w.lane == 0 && w.top > WACC(max_depth)) WACC(max_depth) = w.top;
  __syncwarp();
}

// ================================================================== wide column compression
// Child rows of a wide (4/8/16-word) task are its parent rows restricted to the set bits of
// L' = row(x) and packed (column compression, bit gather).  One row per LANE: the lane loads its
// row's W words and gathers each with the word's precomputed parallel-suffix masks (bits.cuh),
// streaming the packed bits into Wn output words.  cm (shared memory): [5q + i] = mask i of
// word q, [80 + q] = output bit offset of word q; lx = row(x).
__device__ __noinline__ void compress_rows_lanes(const uint32_t* F, const uint32_t* offs, uint32_t n, uint32_t W,
                                                 const uint32_t* lx, const uint32_t* cm, uint32_t Wn, uint32_t* dst,
                                                 int lane) {
  // MBE_COMPRESS_ROWS rows per lane at a time: their word loads are independent (latency overlap)
  for (uint32_t tb = 0; tb < n; tb += 32 * MBE_COMPRESS_ROWS) {
    const uint32_t* src[MBE_COMPRESS_ROWS];
    uint32_t* out[MBE_COMPRESS_ROWS];
    bool ok[MBE_COMPRESS_ROWS];
    uint32_t acc[MBE_COMPRESS_ROWS], accw[MBE_COMPRESS_ROWS];
#pragma unroll
    for (int k = 0; k < MBE_COMPRESS_ROWS; ++k) {
      const uint32_t t = tb + 32 * k + lane;
      ok[k] = t < n;
      src[k] = F + (ok[k] ? offs[t] : 0u);
      out[k] = dst + (size_t)(ok[k] ? t : 0u) * Wn;
      acc[k] = 0u;
      accw[k] = 0u;
    }
#pragma unroll kCompressUnroll
    for (uint32_t q = 0; q < W; ++q) {
      const uint32_t m = lx[q];
      if (m == 0u) continue;  // a zero word of row(x) contributes no column (and no load)
      uint32_t y[MBE_COMPRESS_ROWS];
#pragma unroll
      for (int k = 0; k < MBE_COMPRESS_ROWS; ++k) y[k] = ok[k] ? src[k][q] & m : 0u;
      const uint32_t o = cm[80 + q], d = o >> 5, r = o & 31u;
      const bool spill = r != 0u && r + __popc(m) > 32u;  // spills into the next output word
#pragma unroll
      for (int k = 0; k < MBE_COMPRESS_ROWS; ++k) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          const uint32_t tt = y[k] & cm[5 * q + i];
          y[k] = (y[k] ^ tt) | (tt >> (1 << i));
        }
        if (d > accw[k]) {  // the previous output word is complete
          if (ok[k]) out[k][accw[k]] = acc[k];
          acc[k] = 0;
          accw[k] = d;
        }
        acc[k] |= y[k] << r;
        if (spill) {
          if (ok[k]) out[k][accw[k]] = acc[k];
          acc[k] = y[k] >> (32u - r);
          ++accw[k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < MBE_COMPRESS_ROWS; ++k) {
      if (!ok[k]) continue;
      uint32_t aw = accw[k];
      if (aw < Wn) out[k][aw++] = acc[k];
      for (; aw < Wn; ++aw) out[k][aw] = 0u;
    }
  }
  __syncwarp();
}

// Prepare cm for compress_rows_lanes from row(x) = lx[0..W).
__device__ __forceinline__ void compress_prep_lanes(const uint32_t* lx, uint32_t W, uint32_t* cm, int lane) {
  const uint32_t m = lane < (int)W ? lx[lane] : 0u;
  const uint32_t pc = __popc(m);
  uint32_t incl = pc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane < (int)W) {
    const MbeCompress32 c = mbe_compress_prep(m);
#pragma unroll
    for (int i = 0; i < 5; ++i) cm[5 * lane + i] = c.mv[i];
    cm[80 + lane] = incl - pc;
  }
  __syncwarp();
}

// ================================================================== eager maximality check
// Step 3 for EVERY task of a freshly built bit-row child frame, run once by the
// warp that built it (rows still hot in L1/shared memory) instead of once per scheduled task:
// task t (row r_t, rows in ascending key order) is pruned iff
//   (a) an earlier sibling has an identical row — with ascending keys only an identical row can
//       contain r_t (R2), and identical rows share the key block (key = popc(row)), or
//   (b) some Q row contains r_t.
// ~93% of all tasks end here, so they are never claimed, cached or dispatched.
// Writes the surviving task indices (ascending) to S; returns their number.
#ifndef MBE_QROWS
#define MBE_QROWS 4  // Q rows loaded per step of the eager check (4 beat 6, 8, 16 with the smaller loops: C5 -3 %)
#endif
template <int W>
__device__ __forceinline__ bool prune_q_rows(const Row<W>& r, bool alive, const uint32_t* Qr, uint32_t nQ) {
  for (uint32_t qb = 0; qb < nQ; qb += MBE_QROWS) {
    if (!__any_sync(FULLMASK, alive)) break;
    Row<W> s[MBE_QROWS];
#pragma unroll
    for (int u = 0; u < MBE_QROWS; ++u) s[u] = qb + u < nQ ? load_row<W>(Qr + (size_t)(qb + u) * W) : zero_row<W>();
#pragma unroll
    for (int u = 0; u < MBE_QROWS; ++u)
      if (qb + u < nQ && row_subset<W>(r, s[u])) alive = false;
  }
  return alive;
}

// Row t (ascending key order) is Pr[perm[t] & PERM_IDX] (perm == nullptr: Pr[t]); a set PERM_QDOM bit
// marks a row already found inside a Q' row (prune_q_mark), so the Q scan is skipped (pass nQ = 0).
#define PERM_QDOM 0x80000000u
#define PERM_IDX 0x7fffffffu
template <int W>
__device__ __noinline__ uint32_t prune_frame(const uint32_t* Pr, const uint32_t* perm, uint32_t nP, const uint32_t* Qr,
                                             uint32_t nQ, uint32_t* S, int lane, bool ascending = true) {
  uint32_t nS = 0;
  for (uint32_t tb = 0; tb < nP; tb += 32) {
    const uint32_t t = tb + lane;
    const uint32_t pt = t < nP && perm ? perm[t] : t;
    bool alive = t < nP && !(pt & PERM_QDOM);
    const Row<W> r = alive ? load_row<W>(Pr + (size_t)(pt & PERM_IDX) * W) : zero_row<W>();
    uint32_t key = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) key += __popc(r.w[q]);
    for (int j = (int)t - 1; alive && j >= 0; --j) {
      const Row<W> s = load_row<W>(Pr + (size_t)(perm ? perm[j] & PERM_IDX : (uint32_t)j) * W);
      if (!ascending) {  // order ablation: any earlier sibling may contain row t
        if (row_subset<W>(r, s)) alive = false;
        continue;
      }
      uint32_t kj = 0;
#pragma unroll
      for (int q = 0; q < W; ++q) kj += __popc(s.w[q]);
      if (kj != key) break;
      if (row_eq<W>(r, s)) alive = false;
    }
    alive = prune_q_rows<W>(r, alive, Qr, nQ);
    const uint32_t b = __ballot_sync(FULLMASK, alive);
    if (alive) S[nS + __popc(b & lanemask_lt())] = t;
    nS += __popc(b);
  }
  __syncwarp();
  return nS;
}

// Step 3's Q part on UNSORTED candidates (row idx = Pr[idx]): sets PERM_QDOM in val[idx] for every row
// contained in a Q' row; returns how many are not.  Domination by Q' does not depend on the sibling
// order, so a child whose candidates are all dominated needs no ordering and publishes nothing.
template <int W>
__device__ __noinline__ uint32_t prune_q_mark(const uint32_t* Pr, uint32_t* val, uint32_t nP, const uint32_t* Qr,
                                              uint32_t nQ, int lane) {
  uint32_t n = 0;
  for (uint32_t tb = 0; tb < nP; tb += 32) {
    const uint32_t t = tb + lane;
    const Row<W> r = t < nP ? load_row<W>(Pr + (size_t)t * W) : zero_row<W>();
    const bool alive = prune_q_rows<W>(r, t < nP, Qr, nQ);
    if (t < nP && !alive) val[t] |= PERM_QDOM;
    n += __popc(__ballot_sync(FULLMASK, alive));
  }
  __syncwarp();
  return n;
}

// Wide rows (8/16 words): the same test word-sliced, rows read from memory (L1).  Every row's
// (popcount, OR-fold) metadata is computed once into `meta` (global scratch, >= nP + nQ entries);
// its necessary conditions for == and ⊆ filter the pairs, 8 Q rows in flight per step.
#ifndef MBE_WQROWS
#define MBE_WQROWS 8  // wide eager check: Q-row metadata words loaded per step
#endif
#ifndef MBE_CMASK_MIN
#define MBE_CMASK_MIN 0xffffffffu  // Q rows above which the wide check transposes Q into column masks (with >= 96 P rows)
#endif
__device__ __noinline__ uint32_t prune_frame_wide(const uint32_t* Pr, uint32_t nP, const uint32_t* Qr, uint32_t nQ,
                                                  uint32_t W, uint32_t* S, unsigned long long* meta,
                                                  uint32_t* cmask_buf, int lane, unsigned long long* prof = nullptr,
                                                  bool ascending = true) {
  unsigned long long c0 = prof ? (unsigned long long)clock64() : 0ull, ca = 0, cb = 0;
  for (uint32_t t = lane; t < nP + nQ; t += 32)
    meta[t] = wide_meta(t < nP ? Pr + (size_t)t * W : Qr + (size_t)(t - nP) * W, W);
  __syncwarp();
  if (prof) {
    const unsigned long long c1 = (unsigned long long)clock64();
    prof[0] = c1 - c0;
    c0 = c1;
  }
  const unsigned long long* mq = meta + nP;
  // many Q rows: transpose them once into column masks, cmask[b * G + g] bit i = row 32g + i has
  // column b (one ballot per column per 32 rows)
  const uint32_t G = (nQ + 31) / 32;
  uint32_t* cmask = (nQ > MBE_CMASK_MIN && nP >= 96) ? cmask_buf : nullptr;
  if (cmask) {
    for (uint32_t g = 0; g < G; ++g) {
      const uint32_t i = 32u * g + lane;
      for (uint32_t c = 0; c < W; ++c) {
        const uint32_t wd = i < nQ ? Qr[(size_t)i * W + c] : 0u;
        uint32_t mine = 0;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
          const uint32_t m = __ballot_sync(FULLMASK, (wd >> j) & 1u);
          if (lane == j) mine = m;
        }
        cmask[(size_t)(32u * c + lane) * G + g] = mine;
      }
    }
    __syncwarp();
  }
  uint32_t nS = 0;
  for (uint32_t tb = 0; tb < nP; tb += 32) {
    const uint32_t t = tb + lane;
    bool alive = t < nP;
    const uint32_t* r = Pr + (size_t)(alive ? t : 0u) * W;
    const unsigned long long mr = alive ? meta[t] : 0ull;
    const uint32_t key = (uint32_t)(mr >> MBE_META_SHIFT);
    for (int j = (int)t - 1; alive && j >= 0; --j) {
      const unsigned long long mj = meta[j];
      if (!ascending) {  // order ablation: any earlier sibling may contain row t
        if (meta_may_subset(mr, mj) && wide_subset(r, Pr + (size_t)j * W, W)) alive = false;
        continue;
      }
      if ((uint32_t)(mj >> MBE_META_SHIFT) != key) break;
      if (mj == mr && wide_eq(r, Pr + (size_t)j * W, W)) alive = false;
    }
    if (prof) {
      __syncwarp();
      const unsigned long long c1 = (unsigned long long)clock64();
      ca += c1 - c0;
      c0 = c1;
    }
    if (cmask) {
      // (b) by column masks: the Q rows containing r_t are the AND over the set bits b of r_t of
      // column b's row mask (one word per 32 Q rows, lanes over words)
      uint32_t am = __ballot_sync(FULLMASK, alive);
      while (am) {
        const int sl = __ffs(am) - 1;
        am &= am - 1;
        const uint32_t* rs = Pr + (size_t)(tb + sl) * W;
        bool hit = false;
        for (uint32_t g0 = 0; g0 < G && !hit; g0 += 32) {
          const uint32_t g = g0 + lane;
          uint32_t acc = g < G ? 0xffffffffu : 0u;
          for (uint32_t c = 0; c < W; ++c) {
            uint32_t wd = rs[c];
            while (wd) {
              const uint32_t b = 32u * c + (uint32_t)(__ffs(wd) - 1);
              wd &= wd - 1u;
              if (g < G) acc &= cmask[(size_t)b * G + g];
            }
          }
          hit = __any_sync(FULLMASK, acc != 0u);
        }
        if (hit && lane == sl) alive = false;
      }
    }
    for (uint32_t qb = 0; !cmask && qb < nQ; qb += MBE_WQROWS) {
      if (!__any_sync(FULLMASK, alive)) break;
      unsigned long long m8[MBE_WQROWS];
#pragma unroll
      for (int u = 0; u < MBE_WQROWS; ++u) m8[u] = qb + u < nQ ? mq[qb + u] : ~0ull;
#pragma unroll
      for (int u = 0; u < MBE_WQROWS; ++u)
        if (alive && qb + u < nQ && meta_may_subset(mr, m8[u]) && wide_subset(r, Qr + (size_t)(qb + u) * W, W))
          alive = false;
    }
    if (prof) {
      __syncwarp();
      const unsigned long long c1 = (unsigned long long)clock64();
      cb += c1 - c0;
      c0 = c1;
    }
    const uint32_t b = __ballot_sync(FULLMASK, alive);
    if (alive) S[nS + __popc(b & lanemask_lt())] = t;
    nS += __popc(b);
  }
  __syncwarp();
  if (prof) {
    prof[1] = ca;
    prof[2] = cb;
  }
  return nS;
}

__device__ __forceinline__ uint32_t prune_frame_w(uint32_t W, const uint32_t* Pr, uint32_t nP, const uint32_t* Qr,
                                                  uint32_t nQ, uint32_t* S, unsigned long long* meta,
                                                  uint32_t* cmask_buf, int lane, unsigned long long* prof = nullptr,
                                                  bool ascending = true) {
  __syncwarp();
  if (W == 1) return prune_frame<1>(Pr, nullptr, nP, Qr, nQ, S, lane, ascending);
  if (W == 2) return prune_frame<2>(Pr, nullptr, nP, Qr, nQ, S, lane, ascending);
  if (W == 4) return prune_frame<4>(Pr, nullptr, nP, Qr, nQ, S, lane, ascending);
  return prune_frame_wide(Pr, nP, Qr, nQ, W, S, meta, cmask_buf, lane, prof, ascending);
}

// Account the nP tasks of a child frame decided at build time (nS survive the check).  Algorithmic
// bytes (bit-row path): every task reads row(x) and every row of its frame, i.e.
// 4 W (1 + |P| + |Q|) with |Q| the frame's R1-reduced Q rows (nQ).
__device__ __forceinline__ void account_children(Warp& w, const SearchParams& p, uint32_t nP, uint32_t nS,
                                                 uint32_t W, uint32_t nQ) {
  if (w.lane == 0) {
    WACC(tasks) += nP;
    WACC(pruned) += nP - nS;
    if (MBE_PER_ROOT) {
      atomicAdd(&MBE_PER_ROOT[(size_t)w.cur_root * 4 + 2], (unsigned long long)nP);
      atomicAdd(&MBE_PER_ROOT[(size_t)w.cur_root * 4 + 3], (unsigned long long)(nP - nS));
    }
    if (MBE_STATS_ON) {
      WACC(bitmap_tasks) += nP;
      WACC(ab_bit) += (unsigned long long)nP * 4ull * W * (1ull + nP + nQ);
    }
  }
}

// MBE_STATS only: size of the R1-reduced Q' of a child whose tasks were all decided on the raw
// candidate rows (no frame stored), so its tasks are charged the rows the frame would hold.
__device__ __noinline__ uint32_t stats_r1_size(uint32_t Wn, const uint32_t* src, uint32_t n, Warp& w,
                                               const SearchParams& p) {
  if (n == 0 || (uint64_t)n * Wn > 4ull * p.skey2_off) return n;
  return antichain_w(Wn, src, n, reinterpret_cast<uint32_t*>(WB(skey)), false, w.lane, w.sm);
}

// ================================================================== list path
// Task x on a list frame F (or the implicit root frame when F == nullptr:
// L = V, R = ∅, Q-role = ranks < x, P-role = ranks > x).
__device__ __forceinline__ void list_task(Warp& w, const SearchParams& p, const uint32_t* F, uint32_t i, uint32_t xroot) {
  const DevGraph& g = p.g;
  const int lane = w.lane;
  const bool root = (F == nullptr);
  uint32_t x, nL = 0, nP = 0, nR = 0, key = 0;
  uint64_t sR = 0;
  const uint32_t *L = nullptr, *R = nullptr, *Pid = nullptr;
  if (root) {
    x = xroot;
  } else {
    nL = F[1];
    nP = F[2];
    nR = F[4];
    sR = *reinterpret_cast<const unsigned long long*>(F + 6);
    L = F + MBE_HDR_WORDS;
    R = L + nL;
    Pid = R + nR;
    x = Pid[i];
    key = Pid[nP + i];
  }
  const uint32_t dx = g.offU[x + 1] - g.offU[x];
  const uint32_t* Nx = g.adjU + g.offU[x];

  // twin pre-pruning at the root (R2 at level 1: an earlier vertex with N(v) = N(x))
  if (root && !(p.flags & F_NO_TWIN) && g.twin[x]) {
    account_task(w, p, true);
    if (lane == 0 && MBE_STATS_ON) WACC(list_tasks)++;
    return;
  }

  unsigned long long tph = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
  const unsigned long long tstart = tph;
  unsigned long long tsub[5] = {0, 0, 0, 0, 0};
  unsigned long long tdd[5] = {0, 0, 0, 0, 0};
  unsigned long long pprof[3] = {0, 0, 0};
  // Step 2: L' = L ∩ N(x)
  const uint32_t* Lp;
  uint32_t nLp;
  if (root) {
    Lp = Nx;
    nLp = dx;
  } else {
    nLp = warp_intersect(L, nL, Nx, dx, WB(lbuf), lane);
    Lp = WB(lbuf);
    if (nLp != key) {
      if (lane == 0) set_error(p, 3u, ((unsigned long long)nLp << 32) | key);
      w.failed = true;
      return;
    }
  }
  if (nLp == 0) return;  // reading Z1 (only reachable for a root of degree 0, never enumerated)
  const bool bm = nLp <= p.T;
  const uint32_t Wc = bm ? mbe_words_for(nLp) : 0u;

  // roles of frame rows: tag[v] = (stamp << 32) | (j + 1) for P[j]; TAG_R for R; untagged = Q
  if (!root) {
    w.stamp++;
    const unsigned long long st = ((unsigned long long)w.stamp) << 32;
    for (uint32_t j = lane; j < nP; j += 32)
      *reinterpret_cast<unsigned long long*>(WB(slot) + (size_t)Pid[j] * MBE_SLOT_WORDS + 2) = st | (j + 1);
    for (uint32_t j = lane; j < nR; j += 32)
      *reinterpret_cast<unsigned long long*>(WB(slot) + (size_t)R[j] * MBE_SLOT_WORDS + 2) = st | TAG_R;
    __syncwarp();
  }

  if (MBE_STATS_ON && lane == 0) tsub[0] = (unsigned long long)clock64() - tph;
  MBE_PHASE(6, tph);
  // Reverse scan: for u ∈ L' (position pos), for v ∈ N(u): cnt[v]++,
  // bit pos of row(v) when building a bit-row child.  Flattened over the warp.
  unsigned long long sL = 0;
  uint32_t nt = 0;
  unsigned long long visits = 0;
  for (uint32_t base = 0; base < nLp; base += 32) {
    uint32_t k = base + lane;
    bool kv = k < nLp;
    uint32_t u = kv ? Lp[k] : 0u;
    uint32_t st = kv ? g.offV[u] : 0u;
    uint32_t d = kv ? g.offV[u + 1] - st : 0u;
    if (kv) sL += g.hvV[u];
    uint32_t incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(FULLMASK, incl, 31);
    visits += total;
    // 4 flattened visits per lane per iteration: independent loads/atomics in flight (MLP)
    for (uint32_t fb = 0; fb < total; fb += 32 * MBE_SCAN_MLP) {
      uint32_t vv[MBE_SCAN_MLP], pos[MBE_SCAN_MLP];
      bool fv[MBE_SCAN_MLP];
#pragma unroll
      for (int j = 0; j < MBE_SCAN_MLP; ++j) {
        uint32_t f = fb + 32 * j + lane;
        fv[j] = f < total;
        int lo = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          uint32_t v = __shfl_sync(FULLMASK, incl, lo + s - 1);
          if (v <= f) lo += s;
        }
        uint32_t o_incl = __shfl_sync(FULLMASK, incl, lo);
        uint32_t o_d = __shfl_sync(FULLMASK, d, lo);
        uint32_t o_st = __shfl_sync(FULLMASK, st, lo);
        pos[j] = base + lo;
        vv[j] = fv[j] ? __ldg(&g.adjV[o_st + (f - (o_incl - o_d))]) : 0u;
      }
      uint32_t old[MBE_SCAN_MLP];
#if MBE_INSTR
      if (p.flags & F_NO_RS) {  // noRS ablation: the scan only discovers the vertices (counts below)
#pragma unroll
        for (int j = 0; j < MBE_SCAN_MLP; ++j) old[j] = fv[j] ? atomicExch(&WB(slot)[(size_t)vv[j] * MBE_SLOT_WORDS], 1u) : 1u;
      } else
#endif
      {
#pragma unroll
      for (int j = 0; j < MBE_SCAN_MLP; ++j) old[j] = fv[j] ? atomicAdd(&WB(slot)[(size_t)vv[j] * MBE_SLOT_WORDS], 1u) : 1u;
      }
      // discovery: a vertex's first visit gets the next touched index t; words 0-3 of its bit row live in
      // its slot sector, words 4-15 of a wide row in the candidate-indexed crow[t] (zeroed here; t is
      // recorded in the slot so later visits find it)
      uint32_t tj[MBE_SCAN_MLP];
#pragma unroll
      for (int j = 0; j < MBE_SCAN_MLP; ++j) {
        const bool isnew = old[j] == 0u;
        const uint32_t b = __ballot_sync(FULLMASK, isnew);
        tj[j] = nt + __popc(b & lanemask_lt());
        if (isnew) {
          WB(touched)[tj[j]] = vv[j];
          if (Wc > 4) {
            WB(slot)[(size_t)vv[j] * MBE_SLOT_WORDS + 1] = tj[j] + 1u;
            uint4* cr = reinterpret_cast<uint4*>(WB(crow) + (size_t)tj[j] * MBE_CROW_WORDS);
            for (uint32_t q = 4; q < Wc; q += 4) cr[(q - 4) >> 2] = make_uint4(0u, 0u, 0u, 0u);
          }
        }
        nt += __popc(b);
      }
      if (bm && !(MBE_INSTR && (p.flags & F_NO_RS))) {
#pragma unroll
        for (int j = 0; j < MBE_SCAN_MLP; ++j)
          if (fv[j] && pos[j] < 128u)
            atomicOr(&WB(slot)[(size_t)vv[j] * MBE_SLOT_WORDS + 4 + (pos[j] >> 5)], 1u << (pos[j] & 31));
        if (Wc > 4) {
          // columns >= 128: the row's index comes from this iteration's discoveries (ordered by the
          // __syncwarp) or an earlier one, read from L2
          __syncwarp();
#pragma unroll
          for (int j = 0; j < MBE_SCAN_MLP; ++j)
            if (fv[j] && pos[j] >= 128u) {
              const uint32_t t = old[j] != 0u ? __ldcg(&WB(slot)[(size_t)vv[j] * MBE_SLOT_WORDS + 1]) - 1u : tj[j];
              atomicOr(&WB(crow)[(size_t)t * MBE_CROW_WORDS + (pos[j] >> 5) - 4], 1u << (pos[j] & 31));
            }
        }
      }
    }
  }
  sL = warp_sum64(sL);
  __syncwarp();
#if MBE_INSTR
  if (p.flags & F_NO_RS) {
    // noRS ablation (the paper's "without reverse scanning"): every discovered vertex v
    // gets c = |N(v) ∩ L'| by forward intersection, each element of N(v) binary-searched in the
    // sorted L' (P:138-161 as written), and its bit row from the positions found
    unsigned long long fwd = 0;
    for (uint32_t t = lane; t < nt; t += 32) {
      const uint32_t v = WB(touched)[t];
      const uint32_t* Nv = g.adjU + g.offU[v];
      const uint32_t dv = g.offU[v + 1] - g.offU[v];
      uint32_t c = 0;
      for (uint32_t e = 0; e < dv; ++e) {
        uint32_t lo = 0, hi = nLp;
        const uint32_t y = Nv[e];
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (Lp[mid] < y) lo = mid + 1;
          else hi = mid;
        }
        if (lo < nLp && Lp[lo] == y) {
          ++c;
          if (bm) {
            const uint32_t q = lo >> 5;
            uint32_t* wd = q < 4 ? &WB(slot)[(size_t)v * MBE_SLOT_WORDS + 4 + q] : &WB(crow)[(size_t)t * MBE_CROW_WORDS + q - 4];
            *wd |= 1u << (lo & 31);
          }
        }
      }
      WB(slot)[(size_t)v * MBE_SLOT_WORDS] = c;
      fwd += dv;
    }
    fwd = warp_sum64(fwd);
    __syncwarp();
    if (MBE_STATS_ON && lane == 0) WACC(ab_list) += 4ull * fwd;
  }
#endif

  if (MBE_STATS_ON && lane == 0) tsub[1] = (unsigned long long)clock64() - tph;
  MBE_PHASE(7, tph);
  // Classification of every touched vertex (Steps 3 and 4).
  bool nonmax = false;
  uint32_t nPc = 0, nQc = 0, nRx = 0;
  unsigned long long sRx = 0;
  for (uint32_t tb = 0; tb < nt; tb += 32 * MBE_CLS_MLP) {
    uint32_t vs[MBE_CLS_MLP];
    uint4 sa[MBE_CLS_MLP], sb[MBE_CLS_MLP];
#pragma unroll
    for (int j = 0; j < MBE_CLS_MLP; ++j) {
      uint32_t t = tb + 32 * j + lane;
      vs[j] = t < nt ? WB(touched)[t] : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < MBE_CLS_MLP; ++j) {
      if (vs[j] != 0xffffffffu) {
        const uint4* sp = reinterpret_cast<const uint4*>(WB(slot) + (size_t)vs[j] * MBE_SLOT_WORDS);
        sa[j] = sp[0];
        sb[j] = sp[1];
      } else {
        sa[j] = make_uint4(0u, 0u, 0u, 0u);
        sb[j] = sa[j];
      }
    }
#pragma unroll
    for (int j = 0; j < MBE_CLS_MLP; ++j) {
      if (vs[j] != 0xffffffffu) {
        uint4* sp = reinterpret_cast<uint4*>(WB(slot) + (size_t)vs[j] * MBE_SLOT_WORDS);
        sp[0] = make_uint4(0u, 0u, 0u, 0u);
        sp[1] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int j = 0; j < MBE_CLS_MLP; ++j) {
    const bool valid = vs[j] != 0xffffffffu;
    const uint32_t v = valid ? vs[j] : 0u;
    const uint32_t c = sa[j].x;
    const unsigned long long tg = ((unsigned long long)sa[j].w << 32) | sa[j].z;
    const uint32_t rw[4] = {sb[j].x, sb[j].y, sb[j].z, sb[j].w};
    const uint32_t* crw = WB(crow) + (size_t)(tb + 32 * j + lane) * MBE_CROW_WORDS - 4;  // words 4.. (touched order)
    // role: 0 none/R, 1 Q-role, 2 P-role
    int role = 0;
    if (valid) {
      if (root) {
        role = v == x ? 0 : (v < x ? 1 : 2);
      } else {
        if ((uint32_t)(tg >> 32) == w.stamp) {
          uint32_t info = (uint32_t)tg;
          if (info == TAG_R) role = 0;
          else role = (info - 1 == i) ? 0 : ((info - 1 < i) ? 1 : 2);
        } else {
          role = 1;  // implicit Q: every vertex adjacent to L is in R ∪ P ∪ Q
        }
      }
    }
    bool isQ = role == 1;
    bool isP = role == 2;
    if (isQ && c == nLp) nonmax = true;
    bool isExp = isP && c == nLp;
    bool isPc = isP && c < nLp;
    if (isExp) sRx += g.hvU[v];
    uint32_t be = __ballot_sync(FULLMASK, isExp);
    if (isExp) WB(rbuf)[nRx + __popc(be & lanemask_lt())] = v;
    nRx += __popc(be);
    uint32_t bp = __ballot_sync(FULLMASK, isPc);
    if (isPc) {
      uint32_t idx = nPc + __popc(bp & lanemask_lt());
      WB(skey)[idx] = order_key(p.order, c, v, nLp);
      WB(sval)[idx] = idx;
      if (bm) {
        uint32_t* dst = WB(pbuf) + (size_t)idx * Wc;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          if (q < Wc) dst[q] = rw[q];
        for (uint32_t q = 4; q < Wc; ++q) dst[q] = crw[q];
      }
    }
    nPc += __popc(bp);
    if (bm) {
      uint32_t bq = __ballot_sync(FULLMASK, isQ);
      if (isQ) {
        uint32_t idx = nQc + __popc(bq & lanemask_lt());
        uint32_t* dst = WB(qbuf) + (size_t)idx * Wc;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          if (q < Wc) dst[q] = rw[q];
        for (uint32_t q = 4; q < Wc; ++q) dst[q] = crw[q];
      }
      nQc += __popc(bq);
    }
      }
  }
  nonmax = __any_sync(FULLMASK, nonmax);
  sRx = warp_sum64(sRx);
  __syncwarp();

  if (MBE_STATS_ON && lane == 0) tsub[2] = (unsigned long long)clock64() - tph;
  MBE_PHASE(8, tph);
  account_task(w, p, nonmax);
  if (lane == 0 && MBE_STATS_ON) {
    WACC(list_tasks)++;
    // N(x) + reverse-scan adjacency incl. offsets + touched rows (+ frame L, P, R reads)
    WACC(ab_list) += 4ull * dx + 4ull * (visits + nLp) + 8ull * nt + 4ull * (nL + 2ull * nP + nR);
  }
  if (nonmax) return;

  const uint32_t nRp = nR + 1 + nRx;
  const uint64_t sRp = sR + g.hvU[x] + sRx;
  account_emit(w, p, sL, nLp, sRp, nRp);
  if (MBE_CAP_RECORDS) write_record(w.lane, p, Lp, nLp, R, nR, x, WB(rbuf), nRx);
  if (nPc == 0) return;

  // Child frame (L', R', P' sorted by (count, r), Q') at the arena top.  A wide (8/16-word)
  // bit-row child is built only when its Q' is small (p.wide_qcap) or small relative to the
  // number of sibling tasks that will reuse it (p.wide_ratio), since one warp builds it serially;
  // otherwise the child stays a list frame (implicit Q is exact either way).
  const bool cbm = bm && (Wc <= 4 ? (p.narrow_qmax == 0 || nQc <= p.narrow_qmax || nQc <= p.narrow_ratio * nPc)
                                  : (nQc <= p.wide_qcap || (nQc <= p.wide_ratio * nPc && nQc <= p.wide_qmax)));
  warp_sort_pairs(w, p, nPc, nLp);
  if (MBE_STATS_ON && lane == 0) tsub[3] = (unsigned long long)clock64() - tph;
  MBE_PHASE(9, tph);
  const uint64_t need = MBE_HDR_WORDS + nLp + nRp + 4 + (cbm ? (uint64_t)nPc * (2 + Wc) + (uint64_t)nQc * Wc
                                                            : 2ull * nPc);
  if (!arena_reserve(w, p, need)) return;
  uint32_t* C = WB(arena) + w.atop;
  uint32_t* CL = C + MBE_HDR_WORDS;
  uint32_t* CR = CL + nLp;
  uint32_t* CP = CR + nRp;
  for (uint32_t t = lane; t < nLp; t += 32) CL[t] = Lp[t];
  for (uint32_t t = lane; t < nRp; t += 32) CR[t] = t < nR ? R[t] : (t == nR ? x : WB(rbuf)[t - nR - 1]);
  for (uint32_t t = lane; t < nPc; t += 32) CP[t] = key_id(p.order, WB(skey)[t]);
  uint64_t size;
  uint32_t nQk = 0;
  uint32_t nT = nPc;  // tasks published (bit-row children: the survivors of the eager check)
  bool deferred = false;  // bit-row child published unchecked (HDR_UNCHECKED)
  if (cbm) {
    uint32_t* CPr = WB(arena) + align4(w.atop + (CP + nPc - C));
    for (uint32_t t = lane; t < nPc; t += 32) {
      uint32_t src = WB(sval)[t];
      for (uint32_t q = 0; q < Wc; ++q) CPr[(size_t)t * Wc + q] = WB(pbuf)[(size_t)src * Wc + q];
    }
    uint32_t* CQ = CPr + (size_t)nPc * Wc;
    __syncwarp();
    const uint32_t* qsrc = WB(qbuf);
    uint32_t qn = nQc;
    const unsigned long long td0 = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
    if (MBE_CHAMP_MIN && !(p.flags & F_NO_ANTICHAIN) && Wc <= 8 && nQc > MBE_CHAMP_MIN && nQc <= CHAMP_IDX) {
      qn = champion_filter(WB(qbuf), nQc, Wc, nLp, WB(pbuf), w.sm->hist, lane);  // hist: 256 words >= nLp here
      qsrc = WB(pbuf);
    } else if (!(p.flags & F_NO_ANTICHAIN) && (nQc > p.dedup_min || (Wc >= 8 && nQc > 64))) {  // drop duplicates first
      // hash table in the (now free) sort-key scratch: 4 x cand u64 entries, power of two >= 2 nQc
      uint32_t lg = 1;
      while ((1u << lg) < 2 * nQc) ++lg;
      if ((1ull << lg) <= 4ull * p.skey2_off) {
        qn = dedup_hash_rows(WB(qbuf), nQc, Wc, WB(pbuf), WB(skey), lg, lane);
      } else {
        qn = dedup_sort_rows(WB(qbuf), nQc, Wc, WB(pbuf), WB(skey), WB(sval), WB(skey) + p.skey2_off, WB(sval) + p.skey2_off,
                             w.sm, lane);
      }
      qsrc = WB(pbuf);
    }
    const unsigned long long td1 = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
    // wide rows with many distinct Q' rows: keep the (exactly deduplicated) rows without the
    // O(n * K) antichain pass; extra dominated rows never change a maximality decision
    // The antichain is one warp's serial O(n * K) pass; when Q' is far larger than the number of
    // sibling tasks that will read it, keeping the rows unreduced is cheaper (exact either way).
    const bool keep_all = (p.flags & F_NO_ANTICHAIN) != 0 || (Wc >= 8 && qn > p.wide_acmax) ||
                          (qn > p.ac_min && qn > p.ac_ratio * (nPc + 1));
    bool sorted = false;
    if (!keep_all && Wc <= 4 && qn > 128) {  // descending popcount: the antichain needs no removal pass
      uint32_t* tmp = qsrc == WB(pbuf) ? WB(qbuf) : WB(pbuf);
      popc_sort_rows_desc(qsrc, qn, Wc, tmp, w.sm->hist, lane);  // 32 Wc + 1 <= 129 bins
      qsrc = tmp;
      sorted = true;
    }
    nQk = antichain_w(Wc, qsrc, qn, CQ, keep_all, lane, w.sm, WB(skey), sorted);
    if MBE_STATS_ON {
      tdd[0] = td1 - td0;
      tdd[1] = (unsigned long long)clock64() - td1;
      tdd[2] = qn;
    }
    uint32_t* S = CQ + (size_t)nQk * Wc;  // survivor list of the eager check
    const unsigned long long tp0 = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
    // A large wide child (a hub's level-1 frame) would make its eager check one warp's serial
    // |P'| x |Q'| pass, the critical path of the whole launch on C2/C3: publish every task instead
    // and let each task (spread over warps by stealing) run its own Step 3.
    deferred = Wc >= 8 && p.defer_min && (uint64_t)nPc * nQk >= p.defer_min;
    if (deferred) {
      for (uint32_t t = lane; t < nPc; t += 32) S[t] = t;
      nT = nPc;
    } else {
      nT = prune_frame_w(Wc, CPr, nPc, CQ, nQk, S, WB(skey), WB(pbuf), lane, MBE_STATS_ON ? pprof : nullptr, p.order == 0u);
      account_children(w, p, nPc, nT, Wc, nQk);
    }
    if MBE_STATS_ON {
      tdd[3] = (unsigned long long)clock64() - tp0;
      tdd[4] = td0 - tph;
    }
    size = (uint64_t)(S + nT - C);
  } else {
    uint32_t* CK = CP + nPc;
    for (uint32_t t = lane; t < nPc; t += 32) CK[t] = key_count(p.order, WB(skey)[t], nLp);
    size = (uint64_t)(CK + nPc - C);
  }
  if (nT > 0) {
    if (lane == 0) {
      C[0] = (cbm ? KIND_BITMAP : KIND_LIST) | ((cbm ? Wc : 0u) << 8) | (deferred ? HDR_UNCHECKED : 0u);
      C[1] = nLp;
      C[2] = nPc;
      C[3] = nQk;
      C[4] = nRp;
      C[5] = w.cur_root;
      *reinterpret_cast<unsigned long long*>(C + 6) = sRp;
      if MBE_STATS_ON WACC(ab_write) += 4ull * size;
    }
    publish_frame(w, p, size, nT);
  }
  if (MBE_STATS_ON && lane == 0) tsub[4] = (unsigned long long)clock64() - tph;
  MBE_PHASE(10, tph);
  if (MBE_STATS_ON && lane == 0) {  // diagnostics: remember the longest list task
    const unsigned long long dt = (unsigned long long)clock64() - tstart;
    {
      const uint32_t b = min(11u, (31u - __clz(nt + 1u)) / 2u);
      atomicAdd(&p.gl->list_nt_hist[0][b], 1ull);
      atomicAdd(&p.gl->list_nt_hist[1][b], dt);
    }
    if (atomicMax(&p.gl->longest[0], dt) < dt) {
      unsigned long long* L = p.gl->longest;
      L[1] = root ? 1ull : 0ull; L[2] = x; L[3] = dx; L[4] = nLp; L[5] = nt; L[6] = nPc; L[7] = nQc;
      L[8] = cbm ? Wc : 0ull; L[9] = tsub[0]; L[10] = tsub[1]; L[11] = tsub[2]; L[12] = tsub[3]; L[13] = tsub[4];
      L[14] = nQk; L[15] = nP; L[16] = tdd[0]; L[17] = tdd[1]; L[18] = tdd[2]; L[19] = tdd[3];
      L[20] = tdd[4]; L[21] = pprof[0]; L[22] = pprof[1]; L[23] = pprof[2];
    }
  }
}

// ================================================================== bit-row path
template <int W>
__device__ __forceinline__ void bitmap_task(Warp& w, const SearchParams& p, const uint32_t* F, uint32_t i) {
  const DevGraph& g = p.g;
  const int lane = w.lane;
  const uint32_t nL = F[1], nP = F[2], nQ = F[3], nR = F[4];
  const uint64_t sR = *reinterpret_cast<const unsigned long long*>(F + 6);
  const uint32_t* L = F + MBE_HDR_WORDS;
  const uint32_t* R = L + nL;
  const uint32_t* Pid = R + nR;
  const uint32_t* Prow = F + align4((uint64_t)(Pid + nP - F));
  const uint32_t* Qrow = Prow + (size_t)nP * W;

  unsigned long long tph = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
  const uint32_t x = Pid[i];
  const Row<W> Lx = load_row<W>(Prow + (size_t)i * W);  // L' = row(x) (Step 2)
  uint32_t k = 0;
#pragma unroll
  for (int q = 0; q < W; ++q) k += __popc(Lx.w[q]);

  // Step 3 (maximality) was decided for every task of this frame when it was built
  // (prune_frame): only surviving tasks are ever scheduled, and they were accounted then.
  MBE_PHASE(11, tph);

  // Step 4, expansion over P-role rows j > i.
  const uint32_t Wn = mbe_words_for(k);
  const MbeCompress<W> cmp = mbe_compress_prep_w<W>(Lx.w);
  // 1-word rows: candidate rows are kept as r & row(x) in the frame's columns.  Inclusion, equality and
  // popcount are the same as for the column-compressed rows (compression is a bijection on subsets of
  // row(x)), so Step 3 and R1 decide on them directly; rows are compressed only when a child frame is
  // written (most children are pruned entirely and never need it).
  constexpr bool LAZY = (W == 1);
  uint32_t nPc = 0, nRx = 0, nQc = 0;
  unsigned long long sRx = 0;
  // scratch in shared memory when the candidate bounds fit (P' <= nP-i-1, Q' <= nQ+i)
  const uint32_t maxP = nP - i - 1, maxQ = nQ + i;
  const bool smP = maxP <= MBE_SMEM_SORT && maxP * Wn <= SM_PROW_WORDS && maxP <= SM_RBUF;
  const bool smQ = maxQ * Wn <= SM_QROW_WORDS;
  unsigned long long* kbuf = smP ? w.sm->skey : WB(skey);
  uint32_t* vbuf = smP ? w.sm->sval : WB(sval);
  uint32_t* pbuf = smP ? w.sm->prow : WB(pbuf);
  uint32_t* rbuf = smP ? w.sm->rbuf : WB(rbuf);
  uint32_t* qbuf = smQ ? w.sm->qrow : WB(qbuf);
  uint32_t* lbuf = w.sm->lbuf;
  for (uint32_t jb = i + 1; jb < nP; jb += 32) {
    uint32_t j = jb + lane;
    bool valid = j < nP;
    Row<W> r = valid ? load_row<W>(Prow + (size_t)j * W) : zero_row<W>();
    uint32_t c = row_popc_and<W>(r, Lx);
    uint32_t v = valid ? Pid[j] : 0u;
    bool isExp = valid && c == k;
    bool isPc = valid && c > 0 && c < k;
    if (isExp) sRx += g.hvU[v];
    uint32_t be = __ballot_sync(FULLMASK, isExp);
    if (isExp) rbuf[nRx + __popc(be & lanemask_lt())] = v;
    nRx += __popc(be);
    uint32_t bp = __ballot_sync(FULLMASK, isPc);
    if (isPc) {
      uint32_t idx = nPc + __popc(bp & lanemask_lt());
      kbuf[idx] = order_key(p.order, c, v, k);
      vbuf[idx] = idx;
      if constexpr (LAZY) {
        pbuf[idx] = r.w[0] & Lx.w[0];
      } else {
        uint32_t out[4];
        mbe_compress_apply_w<W>(cmp, r.w, out);
        for (uint32_t q = 0; q < Wn; ++q) pbuf[(size_t)idx * Wn + q] = out[q];
      }
    }
    nPc += __popc(bp);
  }
  sRx = warp_sum64(sRx);
  // sum of hv over L' = L[positions of set bits of row(x)]
  unsigned long long sL = 0;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    uint32_t pos = q * 32 + lane;
    if ((Lx.w[q] >> lane) & 1u) sL += g.hvV[L[pos]];
  }
  sL = warp_sum64(sL);
  const uint32_t nRp = nR + 1 + nRx;
  const uint64_t sRp = sR + g.hvU[x] + sRx;
  account_emit(w, p, sL, k, sRp, nRp);

  MBE_PHASE(12, tph);
  const bool need_child = nPc > 0;
  if (!need_child && !MBE_CAP_RECORDS) return;

  // L' ids in ascending order (L is sorted, positions ascending): into lbuf
#pragma unroll
  for (int q = 0; q < W; ++q) {
    uint32_t bit = (Lx.w[q] >> lane) & 1u;
    uint32_t b = Lx.w[q];
    uint32_t before = 0;
    for (int qq = 0; qq < q; ++qq) before += __popc(Lx.w[qq]);
    if (bit) lbuf[before + __popc(b & lanemask_lt())] = L[q * 32 + lane];
  }
  __syncwarp();
  if (MBE_CAP_RECORDS) write_record(w.lane, p, lbuf, k, R, nR, x, rbuf, nRx);
  if (!need_child) return;

  // Q' candidates: frame Q rows and Q-role siblings P[j<i] meeting L'
  for (uint32_t qb = 0; qb < nQ + i; qb += 32) {
    uint32_t t = qb + lane;
    bool valid = t < nQ + i;
    Row<W> r = zero_row<W>();
    if (valid) r = t < nQ ? load_row<W>(Qrow + (size_t)t * W) : load_row<W>(Prow + (size_t)(t - nQ) * W);
    bool keep = valid && row_any_and<W>(r, Lx);
    uint32_t bq = __ballot_sync(FULLMASK, keep);
    if (keep) {
      uint32_t idx = nQc + __popc(bq & lanemask_lt());
      if constexpr (LAZY) {
        qbuf[idx] = r.w[0] & Lx.w[0];
      } else {
        uint32_t out[4];
        mbe_compress_apply_w<W>(cmp, r.w, out);
        for (uint32_t q = 0; q < Wn; ++q) qbuf[(size_t)idx * Wn + q] = out[q];
      }
    }
    nQc += __popc(bq);
  }
  __syncwarp();
  if (nPc == 1) {
    // The child frame would hold ONE task: x2 = P'[0] with L'' = row'(x2), Q-role = Q', P-role = ∅
    // (Algorithm 1 on a one-element P).  Run it inline instead of building/publishing a frame.
    const uint32_t x2 = key_id(p.order, kbuf[0]);
    uint32_t r2[4] = {0u, 0u, 0u, 0u};
    for (uint32_t q = 0; q < Wn; ++q) r2[q] = pbuf[q];
    bool dom = false;
    for (uint32_t cb = 0; cb < nQc; cb += 32) {
      const uint32_t t = cb + lane;
      bool sup = t < nQc;
      for (uint32_t q = 0; q < Wn && sup; ++q) sup = (r2[q] & ~qbuf[(size_t)t * Wn + q]) == 0u;
      if (__any_sync(FULLMASK, sup)) {
        dom = true;
        break;
      }
    }
    account_task(w, p, dom);
    if MBE_STATS_ON {
      const uint32_t q1 = stats_r1_size(Wn, qbuf, nQc, w, p);
      if (lane == 0) {
        WACC(bitmap_tasks)++;
        WACC(ab_bit) += 4ull * Wn * (2ull + q1);
      }
    }
    if (!dom) {
      if constexpr (LAZY) r2[0] = mbe_compress_apply(cmp.c[0], r2[0]);  // L'' in L' coordinates
      unsigned long long sL2 = 0;
      uint32_t k2 = 0, before = 0;
      for (uint32_t q = 0; q < Wn; ++q) {
        const uint32_t wd = r2[q];
        if ((wd >> lane) & 1u) {
          const uint32_t id = lbuf[q * 32 + lane];
          sL2 += g.hvV[id];
          if (MBE_CAP_RECORDS) WB(touched)[before + __popc(wd & lanemask_lt())] = id;
        }
        before += __popc(wd);
        k2 += __popc(wd);
      }
      sL2 = warp_sum64(sL2);
      account_emit(w, p, sL2, k2, sRp + g.hvU[x2], nRp + 1);
      if (MBE_CAP_RECORDS) {
        if (lane == 0) rbuf[nRx] = x2;
        __syncwarp();
        write_record(w.lane, p, WB(touched), k2, R, nR, x, rbuf, nRx + 1);
      }
    }
    MBE_PHASE(14, tph);
    return;
  }
  // Eager Step 3 for every child task on the scratch rows (raw Q' candidates decide exactly as
  // their antichain does), before anything is written: most children end here with no survivor.
  // The Q' part first, on the unsorted candidates: when it leaves none, no ordering is needed.
  __syncwarp();
  const uint32_t nQa = Wn == 1   ? prune_q_mark<1>(pbuf, vbuf, nPc, qbuf, nQc, lane)
                       : Wn == 2 ? prune_q_mark<2>(pbuf, vbuf, nPc, qbuf, nQc, lane)
                                 : prune_q_mark<4>(pbuf, vbuf, nPc, qbuf, nQc, lane);
  if (nQa == 0) {
    MBE_PHASE(15, tph);
    account_children(w, p, nPc, 0, Wn, MBE_STATS_ON ? stats_r1_size(Wn, qbuf, nQc, w, p) : 0u);
    MBE_PHASE(14, tph);
    return;
  }
  if (smP) sort_pairs_small(kbuf, vbuf, nPc, w.sm, lane);
  else warp_sort_pairs(w, p, nPc, k);
  MBE_PHASE(13, tph);
  // R2 (identical earlier sibling) on the ordered candidates; the Q' decisions ride along in vbuf
  uint32_t* Stmp = WB(touched);
  __syncwarp();
  const bool asc = p.order == 0u;
  const uint32_t nS = Wn == 1   ? prune_frame<1>(pbuf, vbuf, nPc, qbuf, 0u, Stmp, lane, asc)
                      : Wn == 2 ? prune_frame<2>(pbuf, vbuf, nPc, qbuf, 0u, Stmp, lane, asc)
                                : prune_frame<4>(pbuf, vbuf, nPc, qbuf, 0u, Stmp, lane, asc);
  MBE_PHASE(15, tph);
  if (nS == 0) {
    account_children(w, p, nPc, 0, Wn, MBE_STATS_ON ? stats_r1_size(Wn, qbuf, nQc, w, p) : 0u);
    MBE_PHASE(14, tph);
    return;
  }

  const uint64_t need = MBE_HDR_WORDS + k + nRp + 4 + (uint64_t)nPc * (1 + Wn) + (uint64_t)nQc * Wn + nS;
  if (!arena_reserve(w, p, need)) return;
  uint32_t* C = WB(arena) + w.atop;
  uint32_t* CL = C + MBE_HDR_WORDS;
  uint32_t* CR = CL + k;
  uint32_t* CP = CR + nRp;
  for (uint32_t t = lane; t < k; t += 32) CL[t] = lbuf[t];
  for (uint32_t t = lane; t < nRp; t += 32) CR[t] = t < nR ? R[t] : (t == nR ? x : rbuf[t - nR - 1]);
  for (uint32_t t = lane; t < nPc; t += 32) CP[t] = key_id(p.order, kbuf[t]);
  uint32_t* CPr = WB(arena) + align4(w.atop + (CP + nPc - C));
  for (uint32_t t = lane; t < nPc; t += 32) {
    uint32_t src = vbuf[t] & PERM_IDX;
    if constexpr (LAZY) {
      CPr[t] = mbe_compress_apply(cmp.c[0], pbuf[src]);
    } else {
      for (uint32_t q = 0; q < Wn; ++q) CPr[(size_t)t * Wn + q] = pbuf[(size_t)src * Wn + q];
    }
  }
  uint32_t* CQ = CPr + (size_t)nPc * Wn;
  __syncwarp();
  uint32_t nQk;
  if (nQc * Wn <= SM_KEPT_WORDS && !(p.flags & F_NO_ANTICHAIN)) {
    // reduce into shared memory (skey storage is free again), then copy the survivors out
    uint32_t* kept = reinterpret_cast<uint32_t*>(w.sm->skey);
    nQk = antichain_w(Wn, qbuf, nQc, kept, false, lane, w.sm);
    for (uint32_t t = lane; t < nQk * Wn; t += 32) CQ[t] = LAZY ? mbe_compress_apply(cmp.c[0], kept[t]) : kept[t];
  } else {
    nQk = antichain_w(Wn, qbuf, nQc, CQ, (p.flags & F_NO_ANTICHAIN) != 0, lane, w.sm);
    if constexpr (LAZY) {
      for (uint32_t t = lane; t < nQk; t += 32) CQ[t] = mbe_compress_apply(cmp.c[0], CQ[t]);
      __syncwarp();
    }
  }
  account_children(w, p, nPc, nS, Wn, nQk);
  uint32_t* S = CQ + (size_t)nQk * Wn;
  for (uint32_t t = lane; t < nS; t += 32) S[t] = Stmp[t];
  uint64_t size = (uint64_t)(S + nS - C);
  if (lane == 0) {
    C[0] = KIND_BITMAP | (Wn << 8);
    C[1] = k;
    C[2] = nPc;
    C[3] = nQk;
    C[4] = nRp;
    C[5] = w.cur_root;
    *reinterpret_cast<unsigned long long*>(C + 6) = sRp;
    if MBE_STATS_ON WACC(ab_write) += 4ull * size;
  }
  publish_frame(w, p, size, nS);
  MBE_PHASE(14, tph);
}

// ================================================================== wide bit-row path
// Frames with 128 < |L| <= 512 (8 or 16 words per row).  Same steps as
// bitmap_task, word-sliced: row(x) lives in shared memory, every other row is
// streamed from memory (L1) one word at a time, and child rows are column-
// compressed one row per lane (compress_rows_lanes).
__device__ __forceinline__ void bitmap_task_wide(Warp& w, const SearchParams& p, const uint32_t* F, uint32_t i) {
  const DevGraph& g = p.g;
  const int lane = w.lane;
  const uint32_t W = (F[0] >> 8) & 0xffu;
  const uint32_t nL = F[1], nP = F[2], nQ = F[3], nR = F[4];
  const uint64_t sR = *reinterpret_cast<const unsigned long long*>(F + 6);
  const uint32_t* L = F + MBE_HDR_WORDS;
  const uint32_t* R = L + nL;
  const uint32_t* Pid = R + nR;
  const uint32_t* Prow = F + align4((uint64_t)(Pid + nP - F));
  const uint32_t* Qrow = Prow + (size_t)nP * W;
  unsigned long long tph = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;

  const uint32_t x = Pid[i];
  uint32_t* lx = w.sm->lx;
  if (lane < (int)W) lx[lane] = Prow[(size_t)i * W + lane];
  __syncwarp();
  const uint32_t k = __reduce_add_sync(FULLMASK, lane < (int)W ? (uint32_t)__popc(lx[lane]) : 0u);
  // nonzero words of row(x): only they can meet another row (scans below skip the rest)
  const uint32_t nzw = __ballot_sync(FULLMASK, lane < (int)W && lx[lane] != 0u);

  if (F[0] & HDR_UNCHECKED) {
    // Step 3 deferred to the task: x is not maximal iff a Q-role row (frame Q rows and
    // the earlier siblings P[j < i]) contains row(x)
    bool dom = false;
    for (uint32_t tb = 0; tb < nQ + i && !dom; tb += 32) {
      const uint32_t t = tb + lane;
      bool sup = false;
      if (t < nQ + i) {
        const uint32_t* r = t < nQ ? Qrow + (size_t)t * W : Prow + (size_t)(t - nQ) * W;
        sup = true;
        for (uint32_t bb = nzw; bb && sup; bb &= bb - 1u) {
          const uint32_t q = (uint32_t)(__ffs(bb) - 1);
          sup = (lx[q] & ~r[q]) == 0u;
        }
      }
      dom = __any_sync(FULLMASK, sup);
    }
    account_task(w, p, dom);
    if (lane == 0 && MBE_STATS_ON) {
      WACC(bitmap_tasks)++;
      WACC(ab_bit) += 4ull * W * (1ull + nP + nQ);
    }
    if (dom) return;
  }
  // Otherwise Step 3 was decided when the frame was built (prune_frame_wide): this task is maximal.
  MBE_PHASE(11, tph);

  // Step 4: expansion over P-role rows j > i (pbuf keeps the source row index of each P' candidate)
  uint32_t nPc = 0, nRx = 0, nQc = 0;
  unsigned long long sRx = 0;
  for (uint32_t jb = i + 1; jb < nP; jb += 32) {
    const uint32_t j = jb + lane;
    const bool valid = j < nP;
    uint32_t c = 0;
    if (valid) {
      const uint32_t* r = Prow + (size_t)j * W;
      for (uint32_t bb = nzw; bb; bb &= bb - 1u) {
        const uint32_t q = (uint32_t)(__ffs(bb) - 1);
        c += __popc(r[q] & lx[q]);
      }
    }
    const uint32_t v = valid ? Pid[j] : 0u;
    const bool isExp = valid && c == k;
    const bool isPc = valid && c > 0 && c < k;
    if (isExp) sRx += g.hvU[v];
    const uint32_t be = __ballot_sync(FULLMASK, isExp);
    if (isExp) WB(rbuf)[nRx + __popc(be & lanemask_lt())] = v;
    nRx += __popc(be);
    const uint32_t bp = __ballot_sync(FULLMASK, isPc);
    if (isPc) {
      const uint32_t idx = nPc + __popc(bp & lanemask_lt());
      WB(skey)[idx] = order_key(p.order, c, v, k);
      WB(sval)[idx] = idx;
      WB(pbuf)[idx] = j;
    }
    nPc += __popc(bp);
  }
  sRx = warp_sum64(sRx);
  // L' ids and column positions of row(x), in ascending order
  unsigned long long sL = 0;
  uint32_t before = 0;
  for (uint32_t q = 0; q < W; ++q) {
    const uint32_t word = lx[q];
    const bool bit = (word >> lane) & 1u;
    const uint32_t rank = before + __popc(word & lanemask_lt());
    if (bit) {
      const uint32_t id = L[q * 32 + lane];
      sL += g.hvV[id];
      WB(lbuf)[rank] = id;
    }
    before += __popc(word);
  }
  sL = warp_sum64(sL);
  __syncwarp();
  const uint32_t nRp = nR + 1 + nRx;
  const uint64_t sRp = sR + g.hvU[x] + sRx;
  account_emit(w, p, sL, k, sRp, nRp);
  if (MBE_CAP_RECORDS) write_record(w.lane, p, WB(lbuf), k, R, nR, x, WB(rbuf), nRx);
  MBE_PHASE(12, tph);
  if (nPc == 0) return;

  // Q' candidates: Q rows and Q-role siblings P[j<i] meeting L'; qbuf keeps source row pointers
  for (uint32_t qb = 0; qb < nQ + i; qb += 32) {
    const uint32_t t = qb + lane;
    const bool valid = t < nQ + i;
    bool keep = false;
    uint32_t off = 0;
    if (valid) {
      off = t < nQ ? (uint32_t)((Qrow - F) + (size_t)t * W) : (uint32_t)((Prow - F) + (size_t)(t - nQ) * W);
      const uint32_t* r = F + off;
      for (uint32_t bb = nzw; bb && !keep; bb &= bb - 1u) {  // first meeting word decides
        const uint32_t q = (uint32_t)(__ffs(bb) - 1);
        keep = (r[q] & lx[q]) != 0u;
      }
    }
    const uint32_t bq = __ballot_sync(FULLMASK, keep);
    if (keep) WB(qbuf)[nQc + __popc(bq & lanemask_lt())] = off;
    nQc += __popc(bq);
  }
  __syncwarp();
  warp_sort_pairs(w, p, nPc, k);
  MBE_PHASE(13, tph);
  unsigned long long twd = MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
  auto wide_sub = [&](int slot) {  // MBE_STATS diagnostics: wide child-build sub-phases
    if (MBE_STATS_ON && lane == 0) {
      const unsigned long long now = (unsigned long long)clock64();
      atomicAdd(&p.gl->hist[0][slot], 1ull);
      atomicAdd(&p.gl->hist[1][slot], now - twd);
      twd = now;
    }
  };

  const uint32_t Wn = mbe_words_for(k);
  const uint64_t need = MBE_HDR_WORDS + k + nRp + 8 + (uint64_t)nPc * (2 + Wn) + 2ull * nQc * Wn;
  if (!arena_reserve(w, p, need)) return;
  uint32_t* C = WB(arena) + w.atop;
  uint32_t* CL = C + MBE_HDR_WORDS;
  uint32_t* CR = CL + k;
  uint32_t* CP = CR + nRp;
  for (uint32_t t = lane; t < k; t += 32) CL[t] = WB(lbuf)[t];
  for (uint32_t t = lane; t < nRp; t += 32) CR[t] = t < nR ? R[t] : (t == nR ? x : WB(rbuf)[t - nR - 1]);
  for (uint32_t t = lane; t < nPc; t += 32) CP[t] = key_id(p.order, WB(skey)[t]);
  uint32_t* CPr = WB(arena) + align4(w.atop + (CP + nPc - C));
  uint32_t* cm = reinterpret_cast<uint32_t*>(w.sm->posv);  // compression masks (posv is free here)
  compress_prep_lanes(lx, W, cm, lane);
  const uint32_t prow_off = (uint32_t)(Prow - F);
  for (uint32_t t = lane; t < nPc; t += 32) WB(touched)[t] = prow_off + WB(pbuf)[WB(sval)[t]] * W;
  __syncwarp();
  compress_rows_lanes(F, WB(touched), nPc, W, lx, cm, Wn, CPr, lane);
  uint32_t* CQ = CPr + (size_t)nPc * Wn;
  uint32_t* scratch = CQ + (size_t)nQc * Wn;  // compressed Q' candidates, reduced into CQ below
  compress_rows_lanes(F, WB(qbuf), nQc, W, lx, cm, Wn, scratch, lane);
  __syncwarp();
  // eager Step 3 against the raw Q' candidates; the antichain only for frames that survive
  uint32_t* Stmp = WB(touched);
  MBE_PHASE(14, tph);
  wide_sub(29);
  const uint32_t nS = prune_frame_w(Wn, CPr, nPc, scratch, nQc, Stmp, WB(skey), WB(pbuf), lane, nullptr, p.order == 0u);
  MBE_PHASE(15, tph);
  wide_sub(30);
  if (nS == 0) {
    account_children(w, p, nPc, 0, Wn, MBE_STATS_ON ? stats_r1_size(Wn, scratch, nQc, w, p) : 0u);
    MBE_PHASE(14, tph);
    return;
  }
  const uint32_t nQk = antichain_w(Wn, scratch, nQc, CQ, (p.flags & F_NO_ANTICHAIN) != 0, lane, w.sm);
  account_children(w, p, nPc, nS, Wn, nQk);
  wide_sub(31);
  uint32_t* S = CQ + (size_t)nQk * Wn;
  for (uint32_t t = lane; t < nS; t += 32) S[t] = Stmp[t];
  const uint64_t size = (uint64_t)(S + nS - C);
  if (lane == 0) {
    C[0] = KIND_BITMAP | (Wn << 8);
    C[1] = k;
    C[2] = nPc;
    C[3] = nQk;
    C[4] = nRp;
    C[5] = w.cur_root;
    *reinterpret_cast<unsigned long long*>(C + 6) = sRp;
    if MBE_STATS_ON WACC(ab_write) += 4ull * size;
  }
  publish_frame(w, p, size, nS);
  MBE_PHASE(14, tph);
}

__device__ __forceinline__ int task_phase(const uint32_t* F) {
  return (F[0] & 0xffu) == KIND_LIST ? 1 : 2;
}

__device__ __forceinline__ void run_task(Warp& w, const SearchParams& p, const uint32_t* F, uint32_t i,
                                         uint32_t xroot) {
  if (F == nullptr) {  // level-1 subtree of xroot: implicit root frame
    w.cur_root = xroot;
    list_task(w, p, nullptr, 0u, xroot);
    return;
  }
  const uint32_t h = F[0];
  w.cur_root = F[5];
  if ((h & 0xffu) == KIND_LIST) {
    list_task(w, p, F, i, 0u);
  } else {
    const uint32_t W = (h >> 8) & 0xffu;
    // claim index -> row index: the frame's survivor list follows its Q rows
    i = F[align4((uint64_t)MBE_HDR_WORDS + F[1] + F[4] + F[2]) + (size_t)(F[2] + F[3]) * W + i];
    // 1-word rows (the bulk of all tasks) have a register-resident specialisation; wider rows
    // share the word-sliced implementation (one copy of the code: instruction-cache footprint)
    if (W == 1) bitmap_task<1>(w, p, F, i);
#if MBE_NARROW_TEMPLATES & 2
    else if (W == 2) bitmap_task<2>(w, p, F, i);
#endif
#if MBE_NARROW_TEMPLATES & 4
    else if (W == 4) bitmap_task<4>(w, p, F, i);
#endif
    else bitmap_task_wide(w, p, F, i);
  }
}

// Owner batch size from the number of tasks not yet claimed by it (an upper bound).
__device__ __forceinline__ uint32_t claim_batch(uint32_t rem) {
  return rem >= 64u ? 8u : (rem >= 16u ? 4u : (rem >= 6u ? 2u : 1u));
}

__device__ __forceinline__ unsigned long long stats_clock(const SearchParams& p) {
  return MBE_STATS_ON ? (unsigned long long)clock64() : 0ull;
}

// The out-of-line routines below take only the fields they use, by value: taking the address of the
// kernel's SearchParams would force a local-memory copy of it, read back (LDL) on every hot-path use.
struct StealCtx {
  uint32_t n_warps;
  unsigned int* hint;
  unsigned int* tops;
  Desc* desc;
  Globals* gl;
};
struct ClaimCtx {
  Globals* gl;
  unsigned long long* claim_counter;
  unsigned long long* claim_tab;
  uint32_t n_roots, gss_div;
};

// Idle warp: look for a published frame with unclaimed tasks in the warps
// advertised by the hint bitmap, scanning circularly from gw+1,
// and claim ONE task of the bottom-most such frame (largest subtree).
// Returns true with (*victim, *depth, *task) on success.
__device__ __noinline__ bool try_steal(const int lane, const uint32_t gw, const StealCtx p, uint32_t rot,
                                       bool steal_half, uint32_t* victim, uint32_t* depth, uint32_t* task,
                                       uint32_t* task_end) {
  const uint32_t nw = (p.n_warps + 31) >> 5;
  const uint32_t start = ((gw + 1 + rot) % p.n_warps) >> 5;
  int probes = 0;
  for (uint32_t kb = 0; kb < nw && probes < 8; kb += 32) {
    uint32_t k = kb + lane;
    uint32_t word = k < nw ? ld_volatile(&p.hint[(start + k) % nw]) : 0u;
    uint32_t have = __ballot_sync(FULLMASK, word != 0u);
    while (have && probes < 8) {
      int src = __ffs(have) - 1;
      have &= have - 1;
      uint32_t bitsv = __shfl_sync(FULLMASK, word, src);
      uint32_t wi = (start + kb + src) % nw;
      while (bitsv && probes < 8) {
        int b = __ffs(bitsv) - 1;
        bitsv &= bitsv - 1;
        uint32_t v = wi * 32 + b;
        if (v == gw || v >= p.n_warps) continue;
        ++probes;
        for (int attempt = 0; attempt < 2; ++attempt) {
          uint32_t tp = ld_volatile(&p.tops[v]);
          const Desc* vd = p.desc + (size_t)v * MBE_MAXDEPTH;
          int found = -1;
          for (uint32_t db = 0; db < tp && found < 0; db += 32) {
            uint32_t dd = db + lane;
            bool ok = false;
            if (dd < tp && dd < MBE_MAXDEPTH) {
              unsigned long long c = ld_volatile64(&vd[dd].claim);
              ok = (uint32_t)c < (uint32_t)(c >> 32);
            }
            uint32_t bb = __ballot_sync(FULLMASK, ok);
            if (bb) found = (int)(db + __ffs(bb) - 1);
          }
          if (found >= 0) {
            // leave the idle set before claiming, so termination cannot be declared while this
            // warp holds claimed tasks; re-enter it if the claim is lost.  Claim about half of
            // the unclaimed tasks (the range is copied into this warp's own frame).
            unsigned long long old = 0;
            uint32_t k = 1;
            if (lane == 0) {
              unsigned long long* cw = &p.desc[(size_t)v * MBE_MAXDEPTH + found].claim;
              const unsigned long long c = ld_volatile64(cw);
              const uint32_t rem = (uint32_t)(c >> 32) > (uint32_t)c ? (uint32_t)(c >> 32) - (uint32_t)c : 1u;
              k = steal_half ? max(1u, rem / 2) : 1u;
              atomicSub(&p.gl->idle, 1u);
              dbg_delay(2);
              old = atomicAdd(cw, (unsigned long long)k);
              if ((uint32_t)old >= (uint32_t)(old >> 32)) atomicAdd(&p.gl->idle, 1u);
            }
            old = __shfl_sync(FULLMASK, old, 0);
            k = __shfl_sync(FULLMASK, k, 0);
            if ((uint32_t)old < (uint32_t)(old >> 32)) {
              *victim = v;
              *depth = (uint32_t)found;
              *task = (uint32_t)old;
              *task_end = min((uint32_t)old + k, (uint32_t)(old >> 32));
              return true;
            }
          }
          if (attempt == 0) {
            // nothing claimable: clear the hint bit, then re-check once (an owner that published
            // after our scan set the bit before we cleared it, so its frame is visible now)
            if (lane == 0) atomicAnd(&p.hint[v >> 5], ~(1u << (v & 31)));
            __syncwarp();
          }
        }
      }
    }
  }
  return false;
}

// ================================================================== level-1 subtree claims
// Dynamic claiming through a counter shared by every rank ("subtree fetching", lifted to a
// box-wide counter).  The warps of this launch draw LOCAL indices 0, 1, 2, ... from
// gl->lpos; local indices map onto chunks of global root positions that this launch claimed from the
// shared counter with ONE system-scope atomic per chunk (guided self-scheduling: a chunk is
// ceil(remaining / gss_div) positions, so chunks shrink as the list drains).  The chunk table
// (claim_tab, entries (local base << 32) | global start, appended in order) is published through
// gl->claim_state = (chunks << 33) | (done << 32) | local indices covered.  The warp whose local index
// equals the covered count is the only one that claims the next chunk; warps beyond it wait for the
// publication.  The table doubles as the claim log: a relaunch after an arena overflow starts with the
// previous launch's claim_state, so it replays exactly the chunks this call already took.
// Lane 0 only.  Returns the global root position, or ~0u when this rank has no more.
__device__ __noinline__ uint32_t claim_root_shared(const ClaimCtx p) {
  const uint32_t i = atomicAdd(&p.gl->lpos, 1u);
  const uint32_t n = p.n_roots;
  for (;;) {
    const unsigned long long s = ld_volatile64(&p.gl->claim_state);
    const uint32_t known = (uint32_t)s;
    const uint32_t nch = (uint32_t)(s >> 33);
    if (i < known) {  // last chunk whose local base <= i
      uint32_t lo = 0, hi = nch;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint32_t)(ld_volatile64(&p.claim_tab[mid]) >> 32) <= i) lo = mid;
        else hi = mid;
      }
      const unsigned long long e = ld_volatile64(&p.claim_tab[lo]);
      return (uint32_t)e + (i - (uint32_t)(e >> 32));
    }
    if (s & MBE_CLAIM_DONE) return ~0u;
    if (i == known) {  // this warp claims the next chunk for the launch
      const unsigned long long g0 = *(volatile unsigned long long*)p.claim_counter;
      unsigned long long pos = ~0ull, len = 0;
      if (g0 < n) {
        const unsigned long long rem = n - g0;
        const unsigned long long c = (rem + p.gss_div - 1) / p.gss_div;
        dbg_delay(3);
        pos = atomicAdd_system(p.claim_counter, c);
        if (pos < n) len = min(c, (unsigned long long)n - pos);
      }
      if (len == 0) {
        atomicExch(&p.gl->claim_state, s | MBE_CLAIM_DONE);
        return ~0u;
      }
      p.claim_tab[nch] = ((unsigned long long)known << 32) | pos;
      __threadfence();
      atomicExch(&p.gl->claim_state, ((unsigned long long)(nch + 1) << 33) | (known + len));
      continue;
    }
    __nanosleep(128);  // another warp is claiming the chunk that covers i
  }
}

// No-progress watchdog (lane 0): true once no warp has completed a task for p.watchdog_ns.
__device__ __forceinline__ bool watchdog_expired(const SearchParams& p, WarpSmem* sm) {
  if (p.watchdog_ns == 0) return false;
  const unsigned long long pr = ld_volatile64(&p.gl->progress), now = globaltimer_ns();
  if (pr != sm->wd_seen) {
    sm->wd_seen = pr;
    sm->wd_since = now;
    return false;
  }
  return now - sm->wd_since > p.watchdog_ns;
}

// ================================================================== kernel
__global__ void __launch_bounds__(MBE_BLOCK, MBE_MINBLOCKS) mbe_search_kernel(SearchParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib;
  if (gw >= p.n_warps) return;

  Warp w;
  w.lane = lane;
  w.gw = gw;
  uint8_t* base = p.ws + (size_t)gw * p.ws_stride;
  w.base = base;
  w.desc = p.desc + (size_t)gw * MBE_MAXDEPTH;
  w.top = 0;
  w.atop = 0;
  w.stamp = p.stamps[gw];
  w.sm = reinterpret_cast<WarpSmem*>(smem_raw) + wib;
  w.cur_root = 0;
  w.failed = false;
  if (MBE_ACC_SMEM == 0 || lane == 0) {
    WACC(count) = WACC(hash) = WACC(tasks) = WACC(pruned) = WACC(steals) = 0;
    WACC(list_tasks) = WACC(bitmap_tasks) = WACC(frames) = 0;
    WACC(ab_list) = WACC(ab_bit) = WACC(ab_write) = 0;
    WACC(max_depth) = 0;
  }
  if (lane == 0) {
    for (int k = 0; k < 16; ++k) w.sm->ph[k] = 0;
    w.sm->fc_depth = -1;
    w.sm->wd_seen = ~0ull;
    w.sm->wd_since = globaltimer_ns();
  }
  __syncwarp();

  const bool steal = !(p.flags & F_NO_STEAL);
  const unsigned long long t_start = globaltimer_ns();
  const unsigned long long c_start = (unsigned long long)clock64();
  uint32_t done_tasks = 0;
  uint32_t roots = 0;
  bool roots_done = false;
  bool registered = false;
  bool ever_idle = false;
  uint32_t backoff = MBE_BACKOFF_MIN;
  uint32_t rot = 0;

  while (!w.failed) {
    // Pick the next job, then run it at the ONE task call site below (keeps the kernel's
    // instruction footprint small: every task body is inlined exactly once).
    const uint32_t* F = nullptr;  // nullptr: level-1 (root) task of xr
    uint32_t ti = 0, xr = 0, d = 0;
    int kind = 0;                 // 1 owner, 2 root, 3 stolen
    Desc* dsc = nullptr;
    unsigned long long nxt = PEND_NONE;
    unsigned long long t0 = stats_clock(p);
    if (w.top > 0) {
      // ---- owner: next task of the top frame (claims go through the shared cursor so
      // thieves can take siblings; the next claim is prefetched while this task runs)
      d = w.top - 1;
      dsc = &w.desc[d];
      const uint32_t nP = w.sm->fnp[d];
      // owner claims batches of up to 8 tasks per atomic (fewer L2 round trips); unclaimed
      // tasks stay stealable.  The next batch is prefetched while the batch's last task runs.
      uint32_t i = 0;
      if (lane == 0) {
        if (w.sm->bcur[d] < w.sm->bend[d]) {
          i = w.sm->bcur[d]++;
        } else {
          uint32_t old, k;
          if (w.sm->pend[d] != PEND_NONE) {
            old = w.sm->pend[d];
            k = w.sm->pendk[d];
            w.sm->pend[d] = PEND_NONE;
          } else {
            k = claim_batch(nP - min(nP, w.sm->bend[d]));
            old = (uint32_t)atomicAdd(&dsc->claim, (unsigned long long)k);
          }
          i = old;
          w.sm->bcur[d] = old + 1;
          w.sm->bend[d] = min(old + k, nP);
        }
      }
      i = __shfl_sync(FULLMASK, i, 0);
      if (i >= nP) {
        // exhausted: wait for thieves still reading it, then pop
        if (lane == 0) {
          dbg_delay(4);
          while (ld_volatile(&dsc->done) < nP - w.sm->ffirst[d]) {
            if (ld_volatile(&p.gl->error) || watchdog_expired(p, w.sm)) {
              set_error(p, 4u, 1ull);
              w.failed = true;
              break;
            }
            __nanosleep(64);
          }
          atomicExch(&dsc->claim, 0ull);
          dsc->done = 0u;
          p.tops[gw] = d;
          if MBE_STATS_ON w.sm->ph[5] += clock64() - t0;
          if (w.sm->fc_depth == (int)d) w.sm->fc_depth = -1;
        }
        w.failed = __shfl_sync(FULLMASK, (int)w.failed, 0);
        w.top = d;
        w.atop = w.sm->foff[d];
        __syncwarp();
        continue;
      }
      if (lane == 0 && w.sm->bcur[d] >= w.sm->bend[d] && w.sm->bend[d] < nP) {
        const uint32_t k2 = claim_batch(nP - w.sm->bend[d]);
        nxt = atomicAdd(&dsc->claim, (unsigned long long)k2);
        w.sm->pendk[d] = k2;
      }
      F = WB(arena) + w.sm->foff[d];
      const uint32_t fsz = w.sm->fsz[d];
      if (fsz <= FC_WORDS) {
        if (w.sm->fc_depth != (int)d) {  // (re)load the top frame into shared memory
          const uint4* src = reinterpret_cast<const uint4*>(F);
          uint4* dst = reinterpret_cast<uint4*>(w.sm->fcache);
          for (uint32_t t = lane; t < (fsz + 3) / 4; t += 32) dst[t] = src[t];
          __syncwarp();
          if (lane == 0) w.sm->fc_depth = (int)d;
        }
        F = w.sm->fcache;
      }
      ti = i;
      kind = 1;
    } else if (!roots_done) {
      // ---- empty stack: next level-1 subtree (coarse-grained task)
      unsigned long long pos = 0;
      if (lane == 0) {
        if (p.claim_counter) {
          const uint32_t q = claim_root_shared(ClaimCtx{p.gl, p.claim_counter, p.claim_tab, p.g.n_roots, p.gss_div});
          pos = q == ~0u ? ~0ull : q;
        } else {
          dbg_delay(5);
          pos = atomicAdd(&p.gl->root_cursor, 1ull) * p.world + p.rank;
        }
      }
      pos = __shfl_sync(FULLMASK, pos, 0);
      if (pos >= p.g.n_roots) {
        roots_done = true;
        if (lane == 0 && MBE_STATS_ON) atomicMin(&p.gl->t_roots_out, globaltimer_ns() - t_start);
        continue;
      }
      xr = p.g.root_order[pos];
      kind = 2;
      ++roots;
    } else {
      // ---- idle: register, then steal single tasks or terminate
      if (!registered) {
        if (lane == 0) atomicAdd(&p.gl->idle, 1u);
        if (lane == 0 && MBE_STATS_ON && !ever_idle)
          atomicAdd(&p.gl->busy_hist[min(63ull, (globaltimer_ns() - t_start) / 2000000ull)], 1ull);
        ever_idle = true;
        registered = true;
      }
      uint32_t stop = 0;
      if (lane == 0) {
        stop = (ld_volatile(&p.gl->idle) >= p.n_warps) || ld_volatile(&p.gl->error);
        if (!stop && watchdog_expired(p, w.sm)) {
          set_error(p, 4u, 0ull);  // no-progress watchdog: never hang the device
          stop = 1;
        }
      }
      if (__shfl_sync(FULLMASK, stop, 0)) break;
      uint32_t v = 0, vdep = 0, tend = 0;
      bool got = false;
      if (steal) {
        // leaves the idle set only on a successful claim
        got = try_steal(lane, gw, StealCtx{p.n_warps, p.hint, p.tops, p.desc, p.gl}, rot, (p.flags & F_STEAL_HALF) && !(p.flags & F_STEAL_ONE), &v, &vdep, &ti, &tend);
        rot += 97;
      }
      if (!got) {
        if (lane == 0 && MBE_STATS_ON) {
          w.sm->ph[3] += clock64() - t0;
          atomicAdd(&p.gl->tl_hist[3][min(63ull, (globaltimer_ns() - t_start) / 2000000ull)], clock64() - t0);
        }
        unsigned long long t1 = stats_clock(p);
        __nanosleep(backoff);
        if (backoff < MBE_BACKOFF_MAX) backoff <<= 1;
        if (lane == 0 && MBE_STATS_ON) w.sm->ph[4] += clock64() - t1;
        continue;
      }
      backoff = MBE_BACKOFF_MIN;
      registered = false;
      __threadfence();  // acquire: the victim published the frame before its claim word
      if (lane == 0) dbg_delay(6);
      __syncwarp();
      dsc = p.desc + (size_t)v * MBE_MAXDEPTH + vdep;
      const uint32_t off = ld_volatile(&dsc->off);
      F = reinterpret_cast<const uint32_t*>(p.ws + (size_t)v * p.ws_stride + p.o_arena) + off;
      if (tend - ti >= 2) {
        // steal-half: copy the victim's frame into this warp's (empty) arena and publish it as
        // this warp's own frame over the claimed range [ti, tend); then release the victim
        const uint32_t fsz = ld_volatile(&dsc->size);
        if (!arena_reserve(w, p, fsz + 8)) break;
        const uint4* src = reinterpret_cast<const uint4*>(F);
        uint4* dst = reinterpret_cast<uint4*>(WB(arena) + w.atop);
        for (uint32_t t = lane; t < (fsz + 3) / 4; t += 32) dst[t] = src[t];
        __syncwarp();
        if (lane == 0) {
          atomicAdd(&dsc->done, tend - ti);  // the victim no longer needs to wait for this range
          WACC(steals) += tend - ti;
          if MBE_STATS_ON w.sm->ph[3] += clock64() - t0;
        }
        publish_frame(w, p, fsz, tend, ti);
        continue;
      }
      if (lane == 0 && MBE_STATS_ON) {
        const unsigned long long now = clock64();
        w.sm->ph[3] += now - t0;
        t0 = now;
      }
      kind = 3;
    }

    run_task(w, p, F, ti, xr);  // the single task call site

    __syncwarp();
    if (lane == 0) {
      if ((++done_tasks & 255u) == 0u) atomicAdd(&p.gl->progress, 1ull);  // watchdog heartbeat
      if (kind != 2) atomicAdd(&dsc->done, 1u);
      if (kind == 1 && nxt != PEND_NONE) w.sm->pend[d] = (uint32_t)nxt;
      if (kind == 3) WACC(steals)++;
      if MBE_STATS_ON {
        const int ph = kind == 2 ? 0 : task_phase(F);
        const unsigned long long dt = clock64() - t0;
        w.sm->ph[ph] += dt;
        atomicMax(&p.gl->max_task[ph], dt);
        atomicAdd(&p.gl->tl_hist[ph][min(63ull, (globaltimer_ns() - t_start) / 2000000ull)], dt);
        if (ph == 2) {
          const uint32_t b = 31u - __clz(F[2] + F[3] + 1u);
          atomicAdd(&p.gl->hist[0][b], 1ull);
          atomicAdd(&p.gl->hist[1][b], dt);
          const uint32_t bw = 24u + (31u - __clz((F[0] >> 8) & 0xffu));
          atomicAdd(&p.gl->hist[0][bw], 1ull);
          atomicAdd(&p.gl->hist[1][bw], dt);
          if (((F[0] >> 8) & 0xffu) >= 8u) {
            const uint32_t bq = min(7u, (31u - __clz(F[3] + 1u)) / 2u), bp = min(7u, (31u - __clz(F[2] + 1u)) / 2u);
            atomicAdd(&p.gl->wide_hist[0][bq], 1ull);
            atomicAdd(&p.gl->wide_hist[1][bq], dt);
            atomicAdd(&p.gl->wide_hist[2][bp], 1ull);
            atomicAdd(&p.gl->wide_hist[3][bp], dt);
          }
        }
      }
    }
    __syncwarp();
  }

  // flush lane-0 accumulators
  if (lane == 0) {
    if MBE_STATS_ON atomicAdd(&p.gl->exit_hist[min(63ull, (globaltimer_ns() - t_start) / 2000000ull)], 1ull);
    p.stamps[gw] = w.stamp;
    atomicAdd(&p.gl->count, WACC(count));
    atomicAdd(&p.gl->hash, WACC(hash));
    atomicAdd(&p.gl->tasks, WACC(tasks));
    atomicAdd(&p.gl->pruned, WACC(pruned));
    atomicAdd(&p.gl->steals, WACC(steals));
    if (roots) atomicAdd(&p.gl->roots_run, (unsigned long long)roots);
    if MBE_STATS_ON {
      // per-warp workload distribution (Fig. 5 analog): task cycles vs cycles until this warp exits
      const unsigned long long busy = w.sm->ph[0] + w.sm->ph[1] + w.sm->ph[2];
      const unsigned long long total = max(1ull, (unsigned long long)clock64() - c_start);
      atomicAdd(&p.gl->warp_busy_hist[min(19ull, busy * 20ull / total)], 1ull);
      atomicAdd(&p.gl->warp_busy_sum, busy);
      atomicMin(&p.gl->warp_busy_min, busy);
      atomicMax(&p.gl->warp_busy_max, busy);
      atomicAdd(&p.gl->list_tasks, WACC(list_tasks));
      atomicAdd(&p.gl->bitmap_tasks, WACC(bitmap_tasks));
      atomicAdd(&p.gl->frames, WACC(frames));
      atomicAdd(&p.gl->alg_bytes, WACC(ab_list) + WACC(ab_bit) + WACC(ab_write));
      atomicAdd(&p.gl->alg_list, WACC(ab_list));
      atomicAdd(&p.gl->alg_bitrow, WACC(ab_bit));
      atomicAdd(&p.gl->alg_write, WACC(ab_write));
      atomicMax(&p.gl->max_depth, WACC(max_depth));
      for (int k = 0; k < 16; ++k) atomicAdd(&p.gl->phase[k], w.sm->ph[k]);
    }
  }
}

// Twin flags for level-1 pruning (R2 at the root): twin[x] = 1
// iff some vertex of lower rank has exactly N(x).  Lower rank and N(v) ⊇ N(x)
// force equality since deg(v) <= deg(x).  One warp per vertex: candidates are
// the vertices of rank < x and equal degree adjacent to x's lowest-degree
// neighbour u; each is compared element-wise.
__global__ void __launch_bounds__(256) mbe_twin_kernel(DevGraph g, uint8_t* twin) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < g.nU; x += nwarps) {
    const uint32_t ox = g.offU[x], dx = g.offU[x + 1] - ox;
    uint32_t res = 0;
    if (dx > 0) {
      // lowest-degree neighbour of x
      uint32_t best_d = 0xffffffffu, best_u = 0;
      for (uint32_t t = lane; t < dx; t += 32) {
        uint32_t u = g.adjU[ox + t];
        uint32_t du = g.offV[u + 1] - g.offV[u];
        if (du < best_d || (du == best_d && u < best_u)) {
          best_d = du;
          best_u = u;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        uint32_t od = __shfl_xor_sync(FULLMASK, best_d, o), ou = __shfl_xor_sync(FULLMASK, best_u, o);
        if (od < best_d || (od == best_d && ou < best_u)) {
          best_d = od;
          best_u = ou;
        }
      }
      // first rank with degree dx: lower_bound over the non-decreasing degrees
      uint32_t lo = 0, hi = x;
      while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (g.offU[mid + 1] - g.offU[mid] < dx) lo = mid + 1;
        else hi = mid;
      }
      const uint32_t rlo = lo;
      const uint32_t* Nu = g.adjV + g.offV[best_u];
      // candidates v in N(u) with rlo <= v < x
      uint32_t a = 0, b = best_d;
      while (a < b) {
        uint32_t mid = (a + b) >> 1;
        if (Nu[mid] < rlo) a = mid + 1;
        else b = mid;
      }
      for (uint32_t c = a; c < best_d && !res; ++c) {
        uint32_t v = Nu[c];
        if (v >= x) break;
        const uint32_t* Nv = g.adjU + g.offU[v];
        bool diff = false;
        for (uint32_t t = lane; t < dx; t += 32)
          if (Nv[t] != g.adjU[ox + t]) diff = true;
        if (!__any_sync(FULLMASK, diff)) res = 1;
      }
    }
    if (lane == 0) twin[x] = (uint8_t)res;
  }
}

}  // namespace

int MBE_EXPORT(mbe_search_smem_per_warp)() { return (int)sizeof(WarpSmem); }

// Resident CTAs per SM for a launch shape (the persistent kernel needs every CTA co-resident).
int MBE_EXPORT(mbe_search_max_ctas_per_sm)(int block, int smem_bytes) {
  if (cudaFuncSetAttribute(mbe_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)
    return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mbe_search_kernel, block, smem_bytes) != cudaSuccess) return 0;
  return n;
}

int MBE_EXPORT(mbe_launch_search)(const SearchParams& p, int grid, int block, int smem_bytes, void* stream, void* ev0,
                                   void* ev1) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(mbe_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return -1;
    attr_set = true;
  }
  if (cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev0), s) != cudaSuccess) return -1;
  // Cooperative launch: the runtime refuses (instead of deadlocking) when the persistent grid cannot be
  // co-resident, which the idle-count termination requires.
  SearchParams arg = p;
  void* args[] = {&arg};
  if (cudaLaunchCooperativeKernel((const void*)mbe_search_kernel, dim3(grid), dim3(block), args, (size_t)smem_bytes, s) !=
      cudaSuccess)
    return -1;
  return cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev1), s) == cudaSuccess ? 0 : -1;
}

#if !MBE_INSTR
// Root twin flags (graph-only; computed once per loaded side), grid = SMs x 8 CTAs of 8 warps.
int mbe_launch_twin(const DevGraph& g, int sm_count, void* stream) {
  mbe_twin_kernel<<<sm_count * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(g, const_cast<uint8_t*>(g.twin));
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
#endif
