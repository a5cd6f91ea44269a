// mbe_internal.h — device-side data layout shared by the host driver (api.cu)
// and the persistent search kernel (search.cu).  Product code only.
#pragma once
#include <stdint.h>

#ifndef MBE_MAXDEPTH
#define MBE_MAXDEPTH 48    // per-warp stack depth (search depth is 7-11 on C2-C5)
#endif
#define MBE_WMAX 16        // bit rows of up to 16 x 32 = 512 columns
#define MBE_SLOT_WORDS 8   // per-vertex scratch slot: count, touched index + 1, tag (2), bit-row words 0-3 = one 32-B sector
#define MBE_CROW_WORDS 12  // per touched vertex (candidate-indexed): bit-row words 4-15 of wide rows
#ifndef MBE_SMEM_SORT
#define MBE_SMEM_SORT 128  // pairs sorted in shared memory per warp; larger sorts use radix in HBM
#endif
#define MBE_HDR_WORDS 8    // frame header
// Persistent launch shape: 128-thread CTAs, 6 per SM (85 registers/thread, 24 warps/SM).  Early in round 2
// 7 CTAs (72 registers) were 4-5 % faster; once the hot loops were made smaller (scan MLP 2, rolled wide
// compression, 4 Q rows per eager-check step) 6 CTAs measured 1-4 % faster on C3/C5/C5p and equal on C4,
// with 1/7 less workspace (profiles/ab_r2_session2.jsonl); 8 (64 registers) stays slower.
#ifndef MBE_BLOCK
#define MBE_BLOCK 128
#endif
#ifndef MBE_MINBLOCKS
#define MBE_MINBLOCKS 6
#endif

// Relocalization / reduction thresholds (build-time tuning constants; result-invariant).
#define MBE_WIDE_QCAP 256u          // list task -> 8/16-word child if |Q'| <= this ...
#define MBE_WIDE_RATIO 64u          //   ... or |Q'| <= ratio * |P'| (and <= MBE_WIDE_QMAX)
#define MBE_WIDE_QMAX 0xffffffffu
#define MBE_NARROW_QMAX 0u          // same guard for 1/2/4-word children (0 = always relocalize)
#define MBE_NARROW_RATIO 256u
#define MBE_AC_MIN 1024u            // list-path children skip the Q' antichain if |Q'| > AC_MIN and > AC_RATIO (|P'|+1)
#define MBE_AC_RATIO 0xffffffffu
#define MBE_DEDUP_MIN 512u          // Q' candidate sets above this are deduplicated before the antichain
#define MBE_DEFER_MIN_DEFAULT 65536u  // default of mbe_config.defer_min
#define MBE_WIDE_ACMAX 256u         // wide children keep more distinct Q' rows than this unreduced
#define MBE_WATCHDOG_MS_DEFAULT 120000u

// Immutable device graph after ingest.  Candidate side U is
// relabelled by ascending (degree, original id): internal id = rank r(v).
struct DevGraph {
  uint32_t nU, nV;
  uint64_t nE;
  const uint32_t* offU;   // [nU+1]
  const uint32_t* adjU;   // [nE]  U rank -> sorted V ids
  const uint32_t* offV;   // [nV+1]
  const uint32_t* adjV;   // [nE]  V id -> sorted U ranks
  const uint64_t* hvU;    // [nU]  mix64(2*orig + side_bit(U))
  const uint64_t* hvV;    // [nV]  mix64(2*orig + side_bit(V))
  const uint32_t* origU;  // [nU]  rank -> original id
  const uint32_t* root_order;  // [n_roots] execution order of level-1 tasks (cost-descending)
  const uint8_t* twin;    // [nU] 1 if an earlier (lower-rank) vertex has exactly the same neighbourhood
  uint32_t n_roots;
  uint32_t maxdegU;
};

// Published frame descriptor (one per warp per depth).  claim = (nP << 32) | next.
struct Desc {
  unsigned long long claim;  // (task limit << 32) | next unclaimed task
  unsigned int done;         // tasks finished (or handed to a thief's copy) since publication
  unsigned int off;          // word offset of the frame in the owner's arena
  unsigned int size;         // frame size in words
  unsigned int first;        // first task index of this frame's range (copies made by thieves)
  unsigned int pad[2];
};

struct Globals {
  // ---- hot prefix: copied back to the host after every launch (MBE_GLOBALS_HOT_BYTES)
  unsigned long long root_cursor;  // static deal: next local root index
  unsigned int idle;
  unsigned int error;  // 0 ok, 1 arena overflow, 2 depth overflow, 3 internal check, 4 watchdog
  unsigned long long count, hash, tasks, pruned, steals;
  unsigned long long err_info;
  unsigned long long claim_state;  // shared counter: (chunks << 33) | (done << 32) | local indices covered
  unsigned int lpos;               // shared counter: next local root index
  unsigned int pad0;
  unsigned long long progress;     // tasks completed / 256 (no-progress watchdog)
  unsigned long long roots_run;    // level-1 subtrees run by this launch
  unsigned long long out_records, out_ids;
  // ---- MBE_STATS and diagnostics (copied back only when requested)
  unsigned long long list_tasks, bitmap_tasks, frames, alg_bytes;
  unsigned long long alg_list, alg_bitrow, alg_write;  // MBE_STATS: alg_bytes by part
  unsigned int max_depth;
  unsigned int pad;
  unsigned long long phase[16];  // MBE_STATS: Σ over warps of cycles per phase (see mbe.h)
  unsigned long long max_task[4];  // MBE_STATS: longest single task (cycles): root, list, bit-row, -
  unsigned long long t_roots_out;  // MBE_STATS: ns after launch when the level-1 list ran out
  unsigned long long max_phase[16];  // MBE_STATS: longest single occurrence of each sub-phase (cycles)
  unsigned long long longest[24];    // MBE_STATS diagnostics: the longest list-path task (see search.cu)
  unsigned long long hist[2][32];    // MBE_STATS diagnostics: bit-row tasks by log2(|P|+|Q|) of their frame [0, 24) and by
                                     // log2(W) [24, 29): count, cycles
  unsigned long long exit_hist[64];  // MBE_STATS diagnostics: warps by exit time (2 ms buckets after launch)
  unsigned long long tl_hist[4][64];  // MBE_STATS diagnostics: cycles by completion time (2 ms buckets): root, list, bit-row tasks, steal+idle
  unsigned long long busy_hist[64];  // MBE_STATS diagnostics: warps registering idle for the first time, by time
  unsigned long long warp_busy_hist[20];  // MBE_STATS: warps by busy share (Fig. 5 analog), 5 % bins
  unsigned long long warp_busy_sum, warp_busy_min, warp_busy_max;  // MBE_STATS: task cycles per warp
  unsigned long long max_arena_words;  // MBE_STATS: high-water mark of one warp's arena (words)
  unsigned long long list_nt_hist[2][12];  // MBE_STATS diagnostics: list tasks by touched vertices (log4 buckets): count, cycles
  unsigned long long wide_hist[4][8];  // MBE_STATS diagnostics: wide tasks: [0] by log2(nQ) count, [1] cycles, [2] by log2(nP) count, [3] cycles
};
#define MBE_GLOBALS_HOT_BYTES 112
#define MBE_CLAIM_DONE (1ull << 32)

struct SearchParams {
  DevGraph g;
  int cand_side;  // 1 or 2 (A/B orientation of the hash)
  uint32_t T;     // bitmap threshold (<= 32 * MBE_WMAX = 512)
  uint32_t wide_qcap;   // relocalize a list task's child into 8/16-word rows if |Q'| <= wide_qcap
  uint32_t wide_ratio;  //   ... or |Q'| <= wide_ratio * |P'| and |Q'| <= wide_qmax
  uint32_t wide_qmax;
  uint32_t narrow_qmax, narrow_ratio;  // same guard for 1/2/4-word children (narrow_qmax 0 = always)
  uint32_t dedup_min;
  uint32_t defer_min;   // wide list-path children with |P'| * |Q'| >= this defer Step 3 to each task (0 = never)
  uint32_t wide_acmax;  // wide (8/16-word) list-path children keep more distinct Q' rows than this unreduced
  uint32_t ac_min, ac_ratio;  // list-path children skip the antichain if |Q'| > ac_min and > ac_ratio*(|P'|+1)   // list-path children with more Q' candidates are deduplicated before the antichain
  uint32_t flags;
  uint32_t order;  // 0 ascending (default), 1 input, 2 descending (mbe_config.order)
  uint32_t rank, world;
  unsigned long long* claim_counter;  // NULL -> static deal; else shared across ranks (system-scope atomics)
  unsigned long long* claim_tab;      // [n_roots + 1] chunks claimed by this call: (local base << 32) | global start
  uint32_t gss_div;                   // chunk = ceil(remaining / gss_div) (guided self-scheduling, 4 * world)
  uint32_t n_warps;
  unsigned long long watchdog_ns;  // abort (error 4) when no warp completes a task for this long (0: off)
  // per-warp workspace: region w starts at ws + w * ws_stride (bytes); offsets below are bytes
  uint8_t* ws;
  uint64_t ws_stride;
  uint64_t o_slot, o_crow, o_touched, o_lbuf, o_rbuf, o_skey, o_sval, o_pbuf, o_qbuf, o_arena;
  uint64_t skey2_off;  // element offset of the second (ping-pong) sort buffers
  uint64_t arena_words;
  Desc* desc;          // [n_warps * MBE_MAXDEPTH]
  unsigned int* tops;  // [n_warps]
  unsigned int* stamps;  // [n_warps] persistent tag stamps
  unsigned int* hint;    // [ceil(n_warps/32)] bit w set: warp w may hold a frame with unclaimed tasks
  Globals* gl;
  unsigned long long* per_root;  // device [nU*4] or NULL
  // bounded listing (device buffers) or cap_records = 0
  unsigned long long cap_records, cap_ids;
  unsigned long long* rec_off;
  unsigned int* rec_n1;
  unsigned int* rec_n2;
  unsigned int* out_ids;
};

// flags (same values as include/mbe.h)
#define F_NO_STEAL 0x1u
#define F_STATS 0x2u
#define F_NO_ANTICHAIN 0x4u
#define F_NO_TWIN 0x8u
#define F_STEAL_ONE 0x10u
#define F_STEAL_HALF 0x20u
#define F_NO_RS 0x80u

// Launches the twin pre-pass and the persistent search kernel on `stream`;
// ev0/ev1 (cudaEvent_t) bracket the search kernel alone.
int mbe_launch_twin(const DevGraph& g, int sm_count, void* stream);
int mbe_launch_search(const SearchParams& p, int grid, int block, int smem_bytes, void* stream, void* ev0, void* ev1);
int mbe_launch_search_instr(const SearchParams& p, int grid, int block, int smem_bytes, void* stream, void* ev0,
                            void* ev1);
int mbe_search_smem_per_warp();
int mbe_search_max_ctas_per_sm(int block, int smem_bytes);
int mbe_search_smem_per_warp_instr();
int mbe_search_max_ctas_per_sm_instr(int block, int smem_bytes);
