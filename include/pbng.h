/*
 * pbng.h — C ABI of the B200-native PBNG tip-decomposition hot path.
 *
 * Method: Lakhotia, Kannan, Prasanna, "Parallel Peeling of Bipartite Networks
 * for Hierarchical Dense Subgraph Discovery" (arXiv 2110.12511).
 * Citations: "P:n" = line n of the paper text (reference PAPER.md).
 *
 * All compute runs in hand-written sm_100a CUDA kernels (libpbng.so).  No
 * torch types cross this boundary: plain pointers and sizes only.
 *
 * Conventions shared by every entry point
 *   Graph      G(W = (U, V), E), bipartite (Table 1), given as TWO
 *              CSRs of the same edge set:
 *                U.offsets[U.n + 1] (uint64), U.indices[U.m] (uint32 ids in V)
 *                V.offsets[V.n + 1] (uint64), V.indices[V.m] (uint32 ids in U)
 *              offsets[0] = 0, non-decreasing, offsets[n] = m; U.m == V.m;
 *              no duplicate edges; the two CSRs are transposes of each other.
 *              Adjacency order is free: the library relabels both sides by
 *              decreasing degree (Alg.1 l.2-5) into internal sorted
 *              copies and maps results back to the caller's labels.
 *   side       0: peel U (arguments as given); 1: peel V (roles swapped).
 *              "peel side" below means U for side 0 and V for side 1
 *              (tip decomposition peels one vertex set).
 *   Memory     pbng_* (except *_host) take DEVICE pointers for the graph and
 *              the outputs, caller-allocated and caller-owned.  The library
 *              allocates its scratch stream-ordered on `stream` from a private
 *              memory pool per device and frees it before returning; freed
 *              scratch stays mapped in that pool for the next call until
 *              pbng_release_memory() is called.  The device's default memory
 *              pool is not touched.  No other state is kept between calls.
 *   stream     a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Sync       every call returns only after its work on `stream` completed
 *              (the CD loop reads counters back to the host), so outputs are
 *              valid on return.
 *   Errors     PBNG_OK on success.  PBNG_ERR_ARG: null pointer, bad side,
 *              P < 1 or P > PBNG_MAX_P, U.m != V.m, size mismatch.
 *              PBNG_ERR_GRAPH: CSR precondition violated (only detected with
 *              PBNG_OPT_VALIDATE).  PBNG_ERR_OOM: scratch allocation failed.
 *              PBNG_ERR_CUDA: any other CUDA error.  On error output contents
 *              are unspecified; pbng_last_error() returns a thread-local
 *              message.  No exceptions cross the ABI.
 *   Integers   ids uint32 (n < 2^32 - 1), counts / supports / tip numbers
 *              uint64 (tip numbers reach 3e12 in the paper's data).
 */
#ifndef PBNG_H
#define PBNG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBNG_MAX_P 4096u

typedef struct {
  const uint64_t* offsets; /* n + 1 entries */
  const uint32_t* indices; /* m entries */
  uint32_t n;              /* vertices on this side */
  uint64_t m;              /* edges */
} pbng_csr;

/* Work / time counters of one decomposition (filled when stats != NULL).
 * "wedges" = (u, v, u') adjacency entries read, u' = u included. */
typedef struct {
  uint64_t wedges_count;     /* initial butterfly count */
  uint64_t wedges_cd;        /* CD peel iterations + re-counts */
  uint64_t wedges_fd;        /* FD peeling */
  uint64_t support_updates;  /* C(w,2) decrements applied (w >= 2 pairs) */
  uint32_t rho_cd_iters;     /* CD peeling iterations = synchronisation rounds */
  uint32_t recounts;         /* batch re-count branches taken */
  uint32_t partitions_used;  /* <= P (fewer when supports run out) */
  uint32_t fd_rounds_max;    /* most level rounds any FD partition needed */
  float ms_count, ms_cd, ms_fd_build, ms_fd; /* device time per phase */
  uint64_t uv_steps;         /* (u, v) adjacency steps of traversed vertices (all phases) */
  uint64_t uv_steps_fd;      /* ... of which in FD */
  uint64_t updates_fd;       /* support decrements applied in FD (included in support_updates) */
  uint32_t launches;         /* kernels launched by this call */
  uint32_t pad;
  uint64_t impl[4];          /* implementation counters (tier-2 bitmap windows, repeat-table overflows,
                                dense passes) and [3] = CD support decrements that reached partners still
                                live (A_live; counted only with PBNG_OPT_STATS / PBNG_OPT_STATS_DEFER, else 0) */
  /* device time per kernel family, filled only with PBNG_OPT_STATS (CUDA events
   * recorded on `stream` around each launch): index by PBNG_K_* */
  float ms_kernel[16];
  uint64_t impl_hash[4];     /* tier-1 hash aggregation (count + CD): starts, starts split into id-window
                                groups, groups of those starts, starts passed on to the bitmap tier */
} pbng_stats;

enum {
  PBNG_K_INIT = 0,      /* k_init_u / k_init_v / validation */
  PBNG_K_CLASSIFY = 1,  /* k_classify: per-vertex wedge work and tier routing */
  PBNG_K_AGG_WARP = 2,  /* k_agg_warp: tier-0 wedge aggregation (warp per vertex) */
  PBNG_K_AGG_CTA = 3,   /* k_agg_win, k_vp_agg_mid / k_vp_agg_win: CTA-per-start windowed-bitmap tier */
  PBNG_K_AGG_HASH = 4,  /* k_agg_hash / k_vp_agg_hash: CTA-per-start packed-hash tier */
  PBNG_K_SELECT = 5,    /* k_select: frontier selection + compaction */
  PBNG_K_RANGE = 6,     /* k_range_hist: ⋈^init snapshot + range histogram */
  PBNG_K_COMPACT = 7,   /* k_compact*: dynamic deletion */
  PBNG_K_FD_BUILD = 8,  /* partition membership, segments, LPT work */
  PBNG_K_FD = 9,        /* k_fd: persistent fine-grained peeling */
  PBNG_K_COUNT_VP = 10, /* vertex-priority counting kernels (when used) */
  PBNG_K_EDGE = 11,     /* per-edge butterfly counting (k_edge_*) */
  PBNG_K_NUM = 16
};

enum {
  PBNG_OK = 0,
  PBNG_ERR_ARG = 1,
  PBNG_ERR_GRAPH = 2,
  PBNG_ERR_OOM = 3,
  PBNG_ERR_CUDA = 4
};

enum {
  PBNG_OPT_NO_RECOUNT = 1,     /* never take the batch re-count branch (PBNG--) */
  PBNG_OPT_NO_DELETE = 2,      /* no dynamic edge deletion during CD (PBNG-) */
  PBNG_OPT_VALIDATE = 4,       /* O(m) CSR precondition check -> PBNG_ERR_GRAPH */
  PBNG_OPT_STATS = 8,          /* count wedges / updates on device (small overhead) */
  PBNG_OPT_FORCE_RECOUNT = 16, /* test hook: take the re-count branch every CD iteration */
  PBNG_OPT_ONESIDED_COUNT = 32, /* count (and re-count) by one-sided wedge aggregation, W = Σ_v d_v^2
                                   (P:369-373), instead of vertex-priority counting (Alg.1) */
  PBNG_OPT_FD_GRID = 64,        /* test hook: peel every FD partition of <= 4096 members on the whole GPU
                                   (by default only partitions with far above average work) */
  PBNG_OPT_STATS_DEFER = 128    /* like PBNG_OPT_STATS, but the per-kernel-family device times are
                                   summed later by pbng_kernel_times() instead of inside the call */
};

/* Per-vertex butterfly counts of the peel side:
 *   out_support[u] = sum_{u' != u} C(|N_u ∩ N_u'|, 2)   (= ⋈_u, Table 1)
 * computed by vertex-priority counting (Alg.1 pveBcnt, per-vertex part,
 * P:393-426) on the degree-relabeled graph.  out_support: device, peel-side
 * n entries. */
int pbng_count_butterflies(pbng_csr U, pbng_csr V, int side, uint64_t* out_support, void* stream);

/* Per-edge butterfly counts (⋈_e = number of butterflies of G that contain
 * edge e, notation table) by vertex-priority counting, the per-edge
 * part of Alg.1 (pveBcnt; l.27-30: every wedge (mid, last) of a
 * start whose endpoint pair closes c >= 2 wedges adds c - 1 to its two edges).
 *   side               0: out_edge_support[i] is the count of the edge at
 *                      position i of U.indices (row = the U vertex whose
 *                      offsets range holds i); 1: same in V's CSR order.
 *   out_edge_support   device, m entries (uint64).
 *   out_info           HOST array of 4 or NULL: [0] Alg.1 wedges expanded (each
 *                      (start, mid, last) with last ranked above mid and start,
 *                      starts on both sides); [1..3] starts routed to the warp /
 *                      CTA-hash / dense tiers (kernels_edge.cuh).
 * The graph must be simple (no repeated (u, v)); lists need not be sorted.
 * Errors: PBNG_ERR_ARG (null pointers, U.m != V.m), PBNG_ERR_OOM, PBNG_ERR_CUDA.
 * Synchronous: returns after the result is written. */
int pbng_count_edge_butterflies(pbng_csr U, pbng_csr V, int side, uint64_t* out_edge_support,
                                uint64_t* out_info, void* stream);

/* BE-Index (Bloom-Edge-Index), built from the
 * wedges of vertex-priority counting as P:627-634 describes: every pair
 * {start, last} of same-side vertices with c >= 2 common Alg.1 wedges (last
 * ranked above start and above the mids) is the dominant set of a maximal
 * priority bloom with bloom number k_B = c (Definition); its twin
 * edge pairs are ({start, mid}, {mid, last}) for every such mid.
 * Two-call protocol: with bloom_off == NULL only out_sizes is written; then
 * call again with caller-allocated DEVICE arrays of those sizes:
 *   out_sizes   HOST uint64[2]: number of blooms nb, number of twin pairs np
 *   bloom_off   uint64[nb+1]: pairs of bloom b are [bloom_off[b], bloom_off[b+1])
 *   bloom_k     uint32[nb]: bloom number k_B (= bloom_off[b+1] - bloom_off[b])
 *   bloom_dom   uint32[2*nb]: dominant set (x, y) in caller labels, x = the
 *               start, y = last (highest priority); bit 31 of x set when the
 *               dominant set lies in V
 *   pairs       uint32[2*np]: twin pair (e1, e2) as positions in U.indices
 *               (e1 = {start, mid}, e2 = {mid, last})
 * The bloom set depends on the priority order among equal degrees (any
 * order is a valid BE-Index); every butterfly lies in exactly one bloom
 * (Property) and every edge in k_B - 1 butterflies of each bloom
 * holding it (Property).  Errors: PBNG_ERR_ARG, PBNG_ERR_OOM
 * (also when np >= 2^32), PBNG_ERR_CUDA.  Synchronous. */
int pbng_be_index(pbng_csr U, pbng_csr V, uint64_t* out_sizes, uint64_t* bloom_off, uint32_t* bloom_k,
                  uint32_t* bloom_dom, uint32_t* pairs, void* stream);

/* Wing decomposition (wing number θ_e, Definition P:441-449;
 * SURVEY §8(f) f4): BE-Index construction, then level-synchronous peeling of
 * all edges with support <= the current level, with the batch bloom update
 * (a bloom B losing d of its k_B twin pairs in a round takes k_B - 1 from
 * each surviving twin of a lost pair and d from each edge of a kept pair,
 * the update of Alg.3 P:644-674 applied to a batch as P:1452-1490).
 * Exact (the result equals bottom-up peeling, Alg.2).
 *   side        0: out_theta in U.indices order; 1: in V.indices order.
 *   out_theta   device uint64[m].
 *   out_info    HOST uint64[4] or NULL: blooms, twin pairs, level scans,
 *               peeling rounds.
 * Memory: the BE-Index takes about 37 B per twin pair (at most the Alg.1
 * wedges of pbng_count_edge_butterflies); PBNG_ERR_OOM when it does not fit.
 * The paper's CD/FD partitioning of wing decomposition is not
 * used: every level is one global batch.  Errors as above.  Synchronous. */
int pbng_wing_decompose(pbng_csr U, pbng_csr V, int side, uint64_t* out_theta, uint64_t* out_info, void* stream);

/* Tip decomposition of the peel side (tip number θ_u):
 *   count (Alg.1) -> coarse-grained decomposition CD into <= P ranges
 *   (Alg.4 structure P:792-816, tip specialisation P:982-991, adaptive range
 *   P:895-944, batch re-count P:1442-1449, dynamic deletion P:1493-1504)
 *   -> fine-grained decomposition FD of every partition independently on its
 *   induced subgraph G_i with LPT-ordered dynamic
 *   scheduling.
 * out_tip: device, peel-side n entries (θ = 0 for vertices in no butterfly).
 * P: number of partitions, 1 <= P <= PBNG_MAX_P (the paper uses 150).
 * opts: PBNG_OPT_* bit set.  stats: host pointer or NULL. */
int pbng_tip_decompose(pbng_csr U, pbng_csr V, int side, uint32_t P, uint64_t* out_tip,
                       uint32_t opts, pbng_stats* stats, void* stream);

/* Same as pbng_tip_decompose but the CSR arrays (U/V offsets and indices) and
 * out_tip are HOST pointers (pinned memory recommended).  Host->device copies,
 * the decomposition and the device->host copy of θ all run on `stream`
 * inside this call; device buffers are allocated and freed internally. */
int pbng_tip_decompose_host(pbng_csr U, pbng_csr V, int side, uint32_t P, uint64_t* out_tip,
                            uint32_t opts, pbng_stats* stats, void* stream);

/* Test hook: run count + CD only and return the partition plan.
 *   out_part[u]  partition index i in [0, *out_nparts) (device, n entries)
 *   out_init[u]  ⋈^init_u: support of u at the start of its partition
 *                 (device, n entries)
 *   out_bounds   θ(1..P+1) range bounds, HOST array of P + 1 entries:
 *                bounds[0] = 0 < bounds[1] < ... < bounds[nparts] = UINT64_MAX;
 *                entries past nparts are set to UINT64_MAX.
 *   out_nparts   HOST pointer, partitions produced. */
int pbng_tip_plan(pbng_csr U, pbng_csr V, int side, uint32_t P, uint32_t opts, uint32_t* out_part,
                  uint64_t* out_init, uint64_t* out_bounds, uint32_t* out_nparts, void* stream);

/* One level of the k-tip hierarchy, retrieved from tip numbers (P:463-475:
 * tip numbers index "any level of the k-tip hierarchy"; k-tip = Def. 2,
 * P:451-459).  The level is the subgraph induced on U_k = {u : tip[u] >= k}
 * and all of V; its k-tips are the classes of U_k under butterfly
 * connectivity (u ~ u' iff |N_u ∩ N_u'| >= 2, i.e. they share a butterfly,
 * closed transitively: "connected by a series of butterflies").
 *   tip        device, peel-side n entries (normally pbng_tip_decompose's
 *              output; any uint64 vector is accepted and defines U_k).
 *   k          the level; k = 0 keeps every u (vertices in no butterfly are
 *              singleton components); k > max θ gives an empty level.
 *   out_comp   device, peel-side n entries: the smallest id (caller labels)
 *              of u's k-tip, or 0xFFFFFFFF when tip[u] < k.  Labels are
 *              canonical, so results compare bit-exactly.
 *   out_ncomp  HOST pointer: number of k-tips (components) in the level.
 * Computed on the level's subgraph (non-members deleted from the V lists) by
 * the one-sided aggregation tiers in LINK mode: each member u aggregates
 * w(u, u') over partners u' ranked before it and unions with every u' with
 * w >= 2 (lock-free union-find).  Errors as above; PBNG_ERR_ARG for null
 * pointers.  Synchronous like the other entry points. */
int pbng_tip_components(pbng_csr U, pbng_csr V, int side, const uint64_t* tip, uint64_t k, uint32_t* out_comp,
                        uint32_t* out_ncomp, void* stream);

/* Device time per kernel family (ms, indexed by PBNG_K_*) of the last call on
 * this thread made with PBNG_OPT_STATS_DEFER: the call only records a CUDA
 * event pair around each launch on its stream; this function waits for and
 * sums them, so a caller timing the call itself does not pay for the queries.
 * out_ms: host array of PBNG_K_NUM floats.  Returns PBNG_ERR_ARG if out_ms is
 * NULL; all zeros if no deferred call was made since the last query. */
int pbng_kernel_times(float* out_ms);

/* Return the scratch memory the library's private pools keep mapped (on every
 * device used so far) to the driver.  Safe to call at any time when no pbng_*
 * call is running; the next call maps its scratch again. */
int pbng_release_memory(void);

/* Message for the last non-OK return on this thread ("" if none). */
const char* pbng_last_error(void);

/* Library version string, e.g. "pbng-b200 0.1 sm_100a". */
const char* pbng_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PBNG_H */
