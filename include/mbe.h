/* include/mbe.h — C ABI of libmbe: maximal biclique enumeration on B200 (sm_100a).
 *
 * Problem (§II-A): input a bipartite graph G = (U ∪ V, E);
 * output all maximal bicliques, i.e. all pairs (A, B), A ⊆ side 1, B ⊆ side 2,
 * both nonempty, with A × B ⊆ E, A = N(B) and B = N(A) ("a biclique is maximal
 * if it is not a proper subset of any other biclique").
 * Method: the MBEA search of Algorithm 1 with iMBE candidate order
 * (P:234-245), reverse scanning and coarse-grained level-1
 * subtrees with work stealing (§III-C/D), re-designed for sm_100a
 * (see DESIGN.md).  The library reports {count, order-independent 64-bit hash
 * of the canonical (A,B) set}, optionally a bounded listing.
 *
 * Conventions
 *  - Every function returns an int status: MBE_OK (0) or a negative code.  No
 *    exceptions cross the ABI.  On error, *out / *res contents are unspecified
 *    and no handle leaks; mbe_last_error_detail() gives a message.
 *  - Handles are thread-compatible, not re-entrant: do not call two functions
 *    on the same handle concurrently.  Different handles may be used from
 *    different host threads; mbe_load_csr's host->device copies run on an
 *    internal non-blocking stream, so loading the next graph on one thread
 *    overlaps a search running on another (bench.py's streamed e2e).
 *  - No CPU fallback: when no CUDA device is usable, mbe_load_csr returns
 *    MBE_ECUDA.
 */
#ifndef MBE_H_
#define MBE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MBE_OK = 0,
  MBE_EINVAL = -1,    /* bad argument / config (e.g. threads_per_cta not a multiple of 32, world = 0) */
  MBE_ENOMEM = -2,    /* host or device allocation failed */
  MBE_ECUDA = -3,     /* CUDA runtime error or no usable device */
  MBE_EOVERFLOW = -4, /* per-warp frame arena or depth exhausted: result invalid, retry with larger arena_bytes */
  MBE_ERANGE = -5,    /* an edge id >= n2 */
  MBE_EDIST = -6,     /* multi-GPU claim counter unusable */
  MBE_EINTERNAL = -7  /* device-side consistency check failed (a bug; never a silent wrong count) */
};

/* Opaque handle: the graph resident on one device plus the search workspace. */
typedef struct mbe_graph mbe_graph;

/* Load a bipartite graph given as a row-CSR over ORIGINAL 0-based ids:
 *   side 1 = rows (n1 vertices), side 2 = cols (n2 vertices),
 *   row i's neighbours are col_idx[row_ptr[i] .. row_ptr[i+1]).
 * row_ptr: HOST array of n1+1 uint64, row_ptr[0] = 0, non-decreasing (else MBE_EINVAL).
 * col_idx: HOST array of row_ptr[n1] uint32, each < n2 (else MBE_ERANGE).
 * Rows need not be sorted; duplicate edges are allowed and collapse to one
 * (reading Z8); isolated vertices contribute nothing; n1 = 0, n2 = 0 or no
 * edges is a valid empty graph (count 0, hash 0).
 * The caller keeps ownership of both arrays (they are copied before return).
 * device: CUDA ordinal.  flags: bits 0-7 = host ingest threads (0 = auto: min(hardware threads, 16),
 * 1 for small graphs); other bits reserved, pass 0.
 * Ingest builds both CSR directions (sorted, deduplicated),
 * relabels the candidate side by ascending (degree, original id) and uploads
 * everything to device memory owned by the handle. */
int mbe_load_csr(uint32_t n1, uint32_t n2, const uint64_t *row_ptr, const uint32_t *col_idx, int device,
                 uint32_t flags, mbe_graph **out);

/* mbe_config.flags */
#define MBE_NO_STEAL 0x1u     /* disable inter-warp work stealing (result-invariant) */
#define MBE_STATS 0x2u        /* count algorithmic bytes / task kinds (small overhead) */
#define MBE_NO_ANTICHAIN 0x4u /* keep every Q' row instead of the antichain (result-invariant, slower) */
#define MBE_NO_TWIN 0x8u      /* disable root-level twin pre-pruning (result-invariant) */
#define MBE_STEAL_ONE 0x10u   /* thieves take one task at a time (the default since round 1; kept for compatibility) */
#define MBE_STEAL_HALF 0x20u  /* thieves take half of a frame's unclaimed tasks and copy the frame (result-invariant; slower on C2-C5) */
#define MBE_NO_RS 0x80u       /* ablation: counts |N(v) ∩ L'| of list-path tasks by forward intersection instead
                                 of reverse scanning (the paper's noRS; result- and tree-invariant;
                                 runs the instrumented kernel) */
#define MBE_ARENA_GROW 0x40u  /* arena_bytes is the INITIAL per-warp arena: grow it x4 and relaunch on overflow
                                 (always the case when arena_bytes = 0) */

typedef struct {
  uint32_t struct_size;      /* ABI versioning: sizeof(mbe_config) */
  uint32_t ctas_per_sm;      /* persistent CTAs per SM; 0 = auto (6, clamped to the occupancy limit) */
  uint32_t threads_per_cta;  /* multiple of 32, <= 128 (the kernel's launch bound); 0 = auto (128) */
  uint32_t bitmap_threshold; /* frames with |L| <= this use bit rows (<= 512); 0 = auto (largest that fits) */
  int32_t candidate_side;    /* 0 = auto (smaller side, ties: side 1), 1 = rows, 2 = cols; result-invariant */
  uint32_t flags;            /* MBE_* flags above */
  uint32_t rank, world;      /* this process' share of the level-1 subtrees (world >= 1) */
  uint64_t *claim_counter;   /* shared root counter (dynamic claiming), or NULL (static deal:
                                positions k = rank mod world).  Must be mapped on this device and be the
                                same u64 for every rank: mbe_counter_ptr() of an mbe_counter created by one
                                process and opened by the others (CUDA IPC; peer GPUs need P2P/NVLink).  It
                                is advanced with system-scope atomics in chunks of
                                ceil(remaining / (4 * world)) level-1 subtrees (guided self-scheduling); zero
                                it (mbe_counter_reset) before the first rank of a run starts.  Every chunk a
                                call claims is logged, so an arena-overflow relaunch replays exactly its own
                                chunks: no subtree is lost or counted twice. */
  uint64_t arena_bytes;      /* per-warp frame arena; 0 = auto */
  void *stream;              /* cudaStream_t to run on; NULL = the legacy default stream */
  uint64_t *per_root;        /* optional HOST buffer [n_cand][4] = (count, hash, tasks, pruned) of each
                                level-1 subtree, indexed by the candidate side's ORIGINAL id; or NULL */
  uint32_t watchdog_ms;      /* no-progress watchdog: the call fails with MBE_EINTERNAL if no warp completes
                                a task for this long (a hang is never silent).  0 = default (120000);
                                0xffffffff = off.  It is not a limit on total run time. */
  uint32_t defer_min;        /* wide (8/16-word) list-path children with |P'| * |Q'| >= defer_min publish every
                                task with Step 3 deferred to the task (result-invariant); 0 = auto (65536),
                                0xffffffff = never */
  uint32_t order;            /* candidate order (the order ablation; count and hash are
                                order-invariant, the search tree is not): MBE_ORDER_ASCENDING (0, default: the
                                paper's iMBE order: root P by (degree, id), every P' by
                                (|N(v) ∩ L'|, r(v))), MBE_ORDER_INPUT (1: root P by original id, every P' in its
                                parent's order), MBE_ORDER_DESCENDING (2: root P by (-degree, id), every P' by
                                (-|N(v) ∩ L'|, r(v))); r(v) = position in the root order.  Else MBE_EINVAL. */
} mbe_config;
#define MBE_ORDER_ASCENDING 0u
#define MBE_ORDER_INPUT 1u
#define MBE_ORDER_DESCENDING 2u

/* Optional bounded listing; caller-owned HOST buffers.  Record r occupies
 * ids[rec_off[r] .. rec_off[r] + rec_n1[r] + rec_n2[r]): first the side-1 ids
 * (A), then the side-2 ids (B), original ids, each side ascending.  Records
 * come in nondeterministic order. */
typedef struct {
  uint64_t cap_records, cap_ids;
  uint64_t *rec_off;         /* [cap_records] */
  uint32_t *rec_n1, *rec_n2; /* [cap_records] */
  uint32_t *ids;             /* [cap_ids] */
} mbe_output;

typedef struct {
  uint64_t count;           /* # maximal bicliques, both sides nonempty */
  uint64_t hash;            /* Σ H(A,B) mod 2^64 over the result set */
  uint64_t tasks;           /* search-tree nodes: popped candidates x with L' ≠ ∅ */
  uint64_t pruned;          /* tasks rejected by the maximality check (count = tasks - pruned) */
  uint64_t steals;          /* tasks executed by a warp other than the frame's owner */
  uint64_t records_written; /* <= cap_records */
  uint32_t truncated;       /* 1 if the listing overflowed (count/hash still exact) */
  int32_t candidate_side;   /* side actually used (1 or 2) */
  double kernel_ms;         /* device time of the search (CUDA events on the stream) */
  double wall_ms;           /* host time of the whole call */
  uint64_t alg_bytes;       /* MBE_STATS: algorithmic bytes (parts at the end of the struct) */
  uint64_t list_tasks;      /* MBE_STATS: tasks on the list (reverse-scan) path, incl. roots */
  uint64_t bitmap_tasks;    /* MBE_STATS: tasks on the bit-row path */
  uint64_t frames;          /* MBE_STATS: child frames pushed */
  uint32_t n_warps;         /* persistent warps launched */
  uint32_t max_depth;       /* MBE_STATS: deepest stack level reached */
  /* MBE_STATS: Σ over warps of SM cycles spent per phase (the Eq. 1 breakdown, and the
   * fetch/steal/idle shares of Fig. 6).  Totals: [0] level-1 (root) tasks incl. subtree
   * fetch, [1] list-path tasks below level 1, [2] bit-row tasks, [3] stealing (scan + claim),
   * [4] idle backoff, [5] waiting for thieves before a pop.  Sub-phases of list-path tasks (roots
   * included): [6] L' construction + role tags (Eq. 1 "B"), [7] reverse scan, [8] maximality check
   * + expansion classification ("C"+"E"), [9] ordering of P' ("A"), [10] child frame build.
   * Sub-phases of bit-row tasks: [11] maximality check, [12] expansion + emit, [13] Q' rows +
   * ordering, [14] child frame build.  [15] eager maximality check of a bit-row child (prune_frame). */
  uint64_t phase_cycles[16];
  uint64_t max_task_cycles[3]; /* MBE_STATS: longest single task in cycles: [0] level-1, [1] list, [2] bit-row */
  double roots_out_ms;         /* MBE_STATS: time after launch when the level-1 subtree list ran out */
  uint64_t max_phase_cycles[16]; /* MBE_STATS: longest single occurrence of each phase_cycles sub-phase */
  uint64_t roots_claimed;      /* level-1 subtrees this call ran (its share when ranks share a claim counter) */
  uint32_t claim_chunks;       /* chunks it claimed from the shared counter (0 without one) */
  uint32_t attempts;           /* kernel launches: 1 + arena-overflow relaunches */
  /* MBE_STATS: per-warp workload distribution (the Fig. 5 analog): busy_hist[b] = warps whose
   * busy share (cycles in tasks / cycles from launch to the warp's exit) lies in [b/20, (b+1)/20);
   * busy_ms_min/max/mean = cycles in tasks per warp converted at the SM clock. */
  uint32_t busy_hist[20];
  double busy_ms_min, busy_ms_mean, busy_ms_max;
  /* MBE_STATS: alg_bytes = alg_bytes_list + alg_bytes_bitrow + alg_bytes_write:
   * list tasks 4 deg(x) + 4 Σ_{u∈L'}(deg(u)+1) + 8 |touched| + 4 (|L| + 2|P| + |R|); bit-row tasks
   * 4 W (1 + |P| + |Q|) over their frame's stored rows (|Q| R1-reduced); child frames 4 x words written. */
  uint64_t alg_bytes_list, alg_bytes_bitrow, alg_bytes_write;
  uint64_t workspace_bytes;  /* device workspace of the launch (all warps): per warp the frame arena, the
                                candidate buffers sized by max_x |N(N(x))| and the two vertex-indexed tables */
} mbe_result;

/* Enumerate all maximal bicliques of g.  cfg NULL = defaults; res must be
 * non-NULL; out NULL = count + hash only.  Synchronous: returns when the
 * result is on the host.  Result (count, hash) is invariant under every
 * config field except rank/world (which select a share of the level-1
 * subtrees; the shares of all ranks sum to the whole). */
int mbe_enumerate(mbe_graph *g, const mbe_config *cfg, mbe_result *res, mbe_output *out);

/* Canonical text of a bounded listing ("DESIGN DECISIONS":
 * "one biclique per line, `L: id,id,... | R: id,id,...` with original input IDs, lines sorted
 * lexicographically before writing").  Host-only post-processing, no device work.
 *   out       : the mbe_output mbe_enumerate filled (caller-owned HOST buffers, read only).
 *   n_records : records to format, normally res->records_written (<= out->cap_records).
 *   buf, cap  : caller-owned HOST buffer of cap bytes; buf may be NULL when cap = 0 (size query).
 *   *needed   : receives the exact text length in bytes (no NUL terminator is written).
 * Each line is "L: " + the side-1 ids in decimal, comma-separated, in the record's order (ascending)
 * + " | R: " + the side-2 ids likewise + "\n"; the lines are sorted by byte order (strcmp), so the
 * text is identical for every config that enumerates the same set (records arrive unordered).
 * Returns MBE_OK; MBE_EINVAL (NULL pointers, n_records > cap_records, a record outside ids[cap_ids]);
 * MBE_EOVERFLOW if cap < *needed (buf untouched, *needed set); MBE_ENOMEM. */
int mbe_format_listing(const mbe_output *out, uint64_t n_records, char *buf, uint64_t cap, uint64_t *needed);

/* Static description of a loaded graph. */
typedef struct {
  uint32_t n1, n2;
  uint64_t n_edges;       /* after deduplication */
  uint32_t max_deg1, max_deg2;
  int32_t device;
  uint64_t h2d_bytes;     /* bytes copied host -> device by ingest so far */
} mbe_graph_info;
int mbe_get_info(const mbe_graph *g, mbe_graph_info *info);

void mbe_free(mbe_graph *g);             /* NULL-safe; releases the graph's host memory and returns its device
                                            block to a per-process cache reused by the next mbe_load_csr
                                            (no cudaFree, which synchronises the device) */
/* Search workspaces (per-warp scratch + frame arenas) are pooled per device and
 * reused across handles; this frees every pooled workspace not in use and every
 * cached graph block. */
void mbe_release_workspaces(void);
const char *mbe_strerror(int code);      /* static string */

/* Cross-process claim counter for dynamic claiming of level-1 subtrees over several ranks / GPUs
 * (the paper's subtree fetch by atomics, lifted to one counter per box).
 * One process creates it (device memory on its GPU, zeroed), exports the 64-byte CUDA IPC handle, and
 * every other process opens that handle on its own device (a peer GPU needs P2P access, e.g. NVLink;
 * another process on the same GPU also works).  mbe_counter_ptr() is what mbe_config.claim_counter takes.
 * Errors: MBE_EINVAL (NULL arguments), MBE_ECUDA (allocation / IPC / peer mapping failed), MBE_EDIST
 * (opening a handle in the process that created it). */
typedef struct mbe_counter mbe_counter;
int mbe_counter_create(int device, mbe_counter **out);
int mbe_counter_ipc_handle(const mbe_counter *c, void *handle /* 64 bytes, caller-owned */);
int mbe_counter_open(int device, const void *handle /* 64 bytes */, mbe_counter **out);
uint64_t *mbe_counter_ptr(const mbe_counter *c); /* device-visible pointer, NULL if c is NULL */
int mbe_counter_reset(mbe_counter *c, void *stream); /* zero it (stream-ordered; NULL = legacy stream), then sync */
uint64_t mbe_counter_read(mbe_counter *c);          /* current value (synchronous), for diagnostics */
void mbe_counter_close(mbe_counter *c);             /* NULL-safe; unmaps (opened) or frees (created) */
const char *mbe_last_error_detail(void); /* thread-local message of the last failing call */

#ifdef __cplusplus
}
#endif
#endif /* MBE_H_ */
