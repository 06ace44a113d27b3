// pbng.cu — C ABI (include/pbng.h) and host orchestration of the PBNG tip
// decomposition hot path on B200 (sm_100a).
//
// Paper: Lakhotia, Kannan, Prasanna, arXiv 2110.12511 ("P:n" = PAPER.md line).
// Host side only sequences kernels and reads back a few counters per CD
// iteration (the per-iteration barrier the paper counts as ρ);
// every step of the method runs in the kernels of kernels_cd.cuh /
// kernels_fd.cuh.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pbng.h"
#include "kernels_edge.cuh"
#include "kernels_wing.cuh"
#include "kernels_fd.cuh"
#include "kernels_level.cuh"
#include "kernels_relabel.cuh"
#include "kernels_vp.cuh"

#ifndef PBNG_WIN_PRE_MAX
#define PBNG_WIN_PRE_MAX 4096
#endif

using namespace pbng;

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

void check(cudaError_t e, const char* what, int line) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? PBNG_ERR_OOM : PBNG_ERR_CUDA,
         std::string(what) + " (pbng.cu:" + std::to_string(line) + "): " + cudaGetErrorString(e));
  }
}
#define CK(x) check((x), #x, __LINE__)

constexpr uint64_t kInf = ~0ull;

size_t warp_tier_smem() { return (size_t)(kWarpTierThreads / 32) * 2 * kWarpSlots * 4; }
size_t mid_smem() { return sizeof(MidSmem); }
size_t win_smem() { return sizeof(WinSmem); }
size_t hist_smem() { return (size_t)kBins * 12; }
size_t hash_smem() { return sizeof(HashSmem); }
size_t edge_warp_smem() { return (size_t)(kEdgeWarpThreads / 32) * (2 * (1u << kEdgeWarpLog) + kEdgeWarpPb) * 4; }
size_t edge_cta_smem() { return ((size_t)2 * (1u << kEdgeCtaLog) + kEdgeCtaPb) * 4 + sizeof(EdgeCtaScratch); }
size_t edge_dense_smem() { return (size_t)kEdgeDenseWords * 4 + sizeof(EdgeCtaScratch); }
size_t fd_smem() { return ((size_t)(kFdThreads / 32) * 2 * kFdWarpSlots + 2 * kFdCtaSlots + kFdThreads) * 4; }

// Per-device one-time setup: the dynamic shared-memory opt-ins (they apply to
// the current device only) and a private stream-ordered memory pool for the
// library's scratch.  The pool keeps freed scratch mapped, inside a call and
// between calls (re-mapping ~20 GB of config-5 scratch per call costs
// hundreds of ms), until pbng_release_memory() trims it; the device's default
// pool, which other allocators in the process share, is never reconfigured.
constexpr int kMaxDevices = 64;
std::mutex g_dev_mu;
bool g_dev_ready[kMaxDevices];
cudaMemPool_t g_dev_pool[kMaxDevices];

cudaMemPool_t device_setup(int dev) {
  std::lock_guard<std::mutex> lock(g_dev_mu);
  if (dev < 0 || dev >= kMaxDevices) fail(PBNG_ERR_ARG, "device index out of range");
  if (g_dev_ready[dev]) return g_dev_pool[dev];
  {
    cudaMemPoolProps props;
    std::memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    CK(cudaMemPoolCreate(&pool, &props));
    uint64_t thr = ~0ull;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_dev_pool[dev] = pool;
    cudaFuncSetAttribute(k_agg_warp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_mid<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_smem());
    cudaFuncSetAttribute(k_agg_mid<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_smem());
    cudaFuncSetAttribute(k_vp_agg_mid<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_smem());
    cudaFuncSetAttribute(k_vp_agg_mid<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_smem());
    cudaFuncSetAttribute(k_agg_win<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
    cudaFuncSetAttribute(k_agg_win<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
    cudaFuncSetAttribute(k_agg_warp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_mid<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_smem());
    cudaFuncSetAttribute(k_agg_win<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
    cudaFuncSetAttribute(k_agg_lsplit<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
    cudaFuncSetAttribute(k_vp_agg_win<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
    cudaFuncSetAttribute(k_vp_agg_win<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
    cudaFuncSetAttribute(k_vp_agg_warp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_vp_agg_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_range_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist_smem());
    cudaFuncSetAttribute(k_fd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fd_smem());
    cudaFuncSetAttribute(k_fdg_agg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kGridCnt * 4));
    CK(cudaFuncSetAttribute(k_agg_hash<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hash_smem()));
    CK(cudaFuncSetAttribute(k_agg_hash<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hash_smem()));
    CK(cudaFuncSetAttribute(k_agg_hash<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hash_smem()));
    CK(cudaFuncSetAttribute(k_vp_agg_hash, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hash_smem()));
    CK(cudaFuncSetAttribute(k_edge_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_warp_smem()));
    CK(cudaFuncSetAttribute(k_edge_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_cta_smem()));
    CK(cudaFuncSetAttribute(k_edge_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)edge_dense_smem()));
    CK(cudaGetLastError());
  }
  g_dev_ready[dev] = true;
  return g_dev_pool[dev];
}

// Graph oriented so that U is the peel side (device pointers).
struct Dev {
  uint32_t nU, nV;
  uint64_t m;
  const uint64_t* offU;
  const uint32_t* adjU;
  const uint64_t* offV;
  const uint32_t* adjV;
};

std::vector<cudaEvent_t>& event_pool() {
  static thread_local std::vector<cudaEvent_t> pool;
  return pool;
}
cudaEvent_t new_event() {
  std::vector<cudaEvent_t>& pool = event_pool();
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// Per-launch event pairs of the last call made with PBNG_OPT_STATS_DEFER,
// summed by pbng_kernel_times() (so the queries run after the caller's timing).
struct DeferredSpan {
  int kind;
  cudaEvent_t a, b;
};
std::vector<DeferredSpan>& deferred_spans() {
  static thread_local std::vector<DeferredSpan> spans;
  return spans;
}

class Run {
 public:
  explicit Run(cudaStream_t s) : st(s) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    pool = device_setup(dev);
    CK(cudaMallocHost(&hc, sizeof(Counters)));
  }
  ~Run() {
    for (void* p : allocs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    // events go back to a per-thread pool: creating / destroying thousands of
    // events per call (one pair per launch with PBNG_OPT_STATS) costs host time;
    // with deferral the span events are kept for pbng_kernel_times()
    for (cudaEvent_t e : events) event_pool().push_back(e);
    for (const Span& sp : spans) {
      if (defer) {
        deferred_spans().push_back({sp.kind, sp.a, sp.b});
      } else {
        event_pool().push_back(sp.a);
        event_pool().push_back(sp.b);
      }
    }
    if (hc) cudaFreeHost(hc);
    cudaGetLastError();
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, std::max<size_t>(n, 1) * sizeof(T), pool, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(PBNG_ERR_OOM, "cudaMallocAsync of " + std::to_string(n * sizeof(T)) + " bytes failed: " +
                             cudaGetErrorString(e));
    }
    allocs.push_back(p);
    return (T*)p;
  }
  cudaEvent_t event() {
    cudaEvent_t e;
    e = new_event();
    events.push_back(e);
    CK(cudaEventRecord(e, st));
    return e;
  }
  // kernel launch bookkeeping: launch count always; per-family device time
  // (CUDA events on the launch stream) when `timing` is set (PBNG_OPT_STATS)
  void pre(int kind) {
    (void)kind;
    pending = nullptr;
    if (timing) {
      pending = new_event();
      CK(cudaEventRecord(pending, st));
    }
  }
  void post(int kind) {
    check(cudaGetLastError(), "kernel launch", kind);
    launches++;
    if (timing) {
      cudaEvent_t e;
      e = new_event();
      CK(cudaEventRecord(e, st));
      spans.push_back({kind, pending, e});  // span events live in `spans` only
    }
  }
  void kernel_ms(float* out) {
    for (const Span& sp : spans) out[sp.kind] += elapsed_(sp.a, sp.b);
  }
  Counters& readback(Counters* dc) {
    CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return *hc;
  }
  cudaStream_t st;
  cudaMemPool_t pool = nullptr;
  int nsm = 148;
  Counters* hc = nullptr;
  bool timing = false;
  bool defer = false;
  uint32_t launches = 0;

 private:
  struct Span {
    int kind;
    cudaEvent_t a, b;
  };
  static float elapsed_(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
  cudaEvent_t pending = nullptr;
  std::vector<Span> spans;
  std::vector<void*> allocs;
  std::vector<cudaEvent_t> events;
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

void validate(Run& r, const Dev& g) {
  uint32_t* bad = r.alloc<uint32_t>(1);
  CK(cudaMemsetAsync(bad, 0, 4, r.st));
  r.pre(PBNG_K_INIT);
  k_validate_csr<<<r.nsm * 4, 256, 0, r.st>>>(g.nU, g.m, g.offU, g.adjU, g.nV, bad);
  r.post(PBNG_K_INIT);
  r.pre(PBNG_K_INIT);
  k_validate_csr<<<r.nsm * 4, 256, 0, r.st>>>(g.nV, g.m, g.offV, g.adjV, g.nU, bad);
  r.post(PBNG_K_INIT);
  uint32_t hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  if (hb) fail(PBNG_ERR_GRAPH, hb & 1 ? "CSR offsets invalid" : "CSR index out of range");
}

// ---------------------------------------------------------------- relabeling
// Priority relabeling (Alg.1 l.2-5), see kernels_relabel.cuh.
struct SideRank {
  uint32_t n = 0, dmax = 0;
  unsigned long long* binoff = nullptr;  // [dmax + 2]: first rank of degree (dmax - key)
  unsigned long long* edgoff = nullptr;  // [dmax + 2]: first edge of that degree class
  uint32_t* rank = nullptr;              // caller label -> rank
  uint32_t* inv = nullptr;               // rank -> caller label
  uint64_t* offN = nullptr;              // relabeled CSR
  uint32_t* adjN = nullptr;
  uint32_t n_gt_small = 0, n_gt_tile = 0, n_gt_fill = 0;  // lists longer than 32 / 4096 / 2048
};

void scan_u64(Run& r, unsigned long long* a, uint64_t n) {
  if (!n) return;
  const uint64_t nt = (n + kScanTile - 1) / kScanTile;
  uint64_t* ts = r.alloc<uint64_t>(nt);
  r.pre(PBNG_K_INIT);
  k_scan_tiles<<<(unsigned)nt, kScanThreads, 0, r.st>>>(n, (uint64_t*)a, ts);
  r.post(PBNG_K_INIT);
  r.pre(PBNG_K_INIT);
  k_scan_top<<<1, kScanThreads, 0, r.st>>>((uint32_t)nt, ts);
  r.post(PBNG_K_INIT);
  r.pre(PBNG_K_INIT);
  k_scan_add<<<r.nsm * 4, 256, 0, r.st>>>(n, (uint64_t*)a, ts);
  r.post(PBNG_K_INIT);
}

uint64_t read_u64(Run& r, const unsigned long long* p) {
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, p, 8, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  return h;
}

void rank_side(Run& r, uint32_t n, uint64_t m, const uint64_t* off, SideRank& s) {
  s.n = n;
  unsigned long long* dm = r.alloc<unsigned long long>(1);
  CK(cudaMemsetAsync(dm, 0, 8, r.st));
  r.pre(PBNG_K_INIT);
  k_deg_max<<<r.nsm * 4, 256, 0, r.st>>>(n, off, dm);
  r.post(PBNG_K_INIT);
  s.dmax = (uint32_t)read_u64(r, dm);
  const uint64_t nb = (uint64_t)s.dmax + 2;
  s.binoff = r.alloc<unsigned long long>(nb);
  s.edgoff = r.alloc<unsigned long long>(nb);
  uint32_t* cursor = r.alloc<uint32_t>(nb);
  CK(cudaMemsetAsync(s.binoff, 0, nb * 8, r.st));
  CK(cudaMemsetAsync(s.edgoff, 0, nb * 8, r.st));
  CK(cudaMemsetAsync(cursor, 0, nb * 4, r.st));
  r.pre(PBNG_K_INIT);
  k_deg_hist<<<r.nsm * 8, 256, 0, r.st>>>(n, off, s.dmax, s.binoff, s.edgoff);
  r.post(PBNG_K_INIT);
  scan_u64(r, s.binoff, nb);
  scan_u64(r, s.edgoff, nb);
  s.rank = r.alloc<uint32_t>(n);
  s.inv = r.alloc<uint32_t>(n);
  s.offN = r.alloc<uint64_t>((size_t)n + 1);
  r.pre(PBNG_K_INIT);
  k_rank_scatter<<<r.nsm * 8, 256, 0, r.st>>>(n, off, s.dmax, s.binoff, cursor, s.rank, s.inv);
  r.post(PBNG_K_INIT);
  r.pre(PBNG_K_INIT);
  k_rank_offsets<<<r.nsm * 8, 256, 0, r.st>>>(n, m, s.inv, off, s.dmax, s.binoff, s.edgoff, s.offN);
  r.post(PBNG_K_INIT);
  s.adjN = r.alloc<uint32_t>(m);
  // number of lists longer than d: binoff[dmax - d] (d < dmax), else 0
  auto n_gt = [&](uint32_t d) -> uint32_t { return d < s.dmax ? (uint32_t)read_u64(r, s.binoff + (s.dmax - d)) : 0u; };
  s.n_gt_small = n_gt(kSortSmall);
  s.n_gt_tile = n_gt(kSortTile);
  s.n_gt_fill = n_gt(2048);
}

void fill_side(Run& r, const uint64_t* off, const uint32_t* adj, const SideRank& s, const uint32_t* rank_other) {
  if (!s.n) return;
  r.pre(PBNG_K_INIT);
  k_relabel_fill<<<r.nsm * 8, 256, 0, r.st>>>(s.n, s.n_gt_fill, s.inv, off, adj, s.offN, rank_other, s.adjN);
  r.post(PBNG_K_INIT);
  if (s.n_gt_fill) {
    r.pre(PBNG_K_INIT);
    k_relabel_fill_big<<<std::min<uint32_t>(s.n_gt_fill, r.nsm * 4), 512, 0, r.st>>>(s.n_gt_fill, s.inv, off, adj,
                                                                                     s.offN, rank_other, s.adjN);
    r.post(PBNG_K_INIT);
  }
}

void sort_side(Run& r, const SideRank& s, uint32_t* tmp) {
  if (!s.n) return;
  if (s.n > s.n_gt_small) {
    r.pre(PBNG_K_INIT);
    k_sort_small<<<r.nsm * 8, 256, 0, r.st>>>(s.n_gt_small, s.n, s.offN, s.adjN);
    r.post(PBNG_K_INIT);
  }
  // lists longer than one tile: chunk tasks, then merge passes
  std::vector<uint64_t> hoff(s.n_gt_tile + 1);
  std::vector<ulonglong2> chunks;
  if (s.n_gt_tile) {
    CK(cudaMemcpyAsync(hoff.data(), s.offN, hoff.size() * 8, cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    for (uint32_t i = 0; i < s.n_gt_tile; i++)
      for (uint64_t a = hoff[i]; a < hoff[i + 1]; a += kSortTile)
        chunks.push_back(make_ulonglong2(a, std::min<uint64_t>(kSortTile, hoff[i + 1] - a)));
  }
  ulonglong2* dch = r.alloc<ulonglong2>(chunks.size());
  if (!chunks.empty())
    CK(cudaMemcpyAsync(dch, chunks.data(), chunks.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice, r.st));
  const uint32_t nseg = (s.n_gt_small - s.n_gt_tile) + (uint32_t)chunks.size();
  if (nseg) {
    r.pre(PBNG_K_INIT);
    k_sort_tile<<<std::min<uint32_t>(nseg, r.nsm * 4), kSortThreads, 0, r.st>>>(
        s.n_gt_tile, s.n_gt_small, s.offN, dch, (uint32_t)chunks.size(), s.adjN);
    r.post(PBNG_K_INIT);
  }
  for (uint64_t run = kSortTile;; run *= 2) {
    std::vector<ulonglong2> tiles;
    for (uint32_t i = 0; i < s.n_gt_tile; i++) {
      const uint64_t len = hoff[i + 1] - hoff[i];
      if (len <= run) continue;
      for (uint64_t t = 0; t * kSortTile < len; t++) tiles.push_back(make_ulonglong2(hoff[i], len | (t << 32)));
    }
    if (tiles.empty()) break;
    ulonglong2* dt = r.alloc<ulonglong2>(tiles.size());
    CK(cudaMemcpyAsync(dt, tiles.data(), tiles.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice, r.st));
    const uint32_t nt = (uint32_t)tiles.size();
    r.pre(PBNG_K_INIT);
    k_merge_pass<<<std::min<uint32_t>(nt, r.nsm * 4), kSortThreads, 0, r.st>>>(dt, nt, run, s.adjN, tmp);
    r.post(PBNG_K_INIT);
    r.pre(PBNG_K_INIT);
    k_copy_tiles<<<std::min<uint32_t>(nt, r.nsm * 4), 512, 0, r.st>>>(dt, nt, tmp, s.adjN);
    r.post(PBNG_K_INIT);
    CK(cudaStreamSynchronize(r.st));  // host vector `tiles` must outlive the copy
  }
}

// Relabel both sides of g; returns the graph in rank labels (sorted lists).
Dev relabel(Run& r, const Dev& g, SideRank& RU, SideRank& RV) {
  rank_side(r, g.nU, g.m, g.offU, RU);
  rank_side(r, g.nV, g.m, g.offV, RV);
  if (g.m) {
    fill_side(r, g.offU, g.adjU, RU, RV.rank);
    fill_side(r, g.offV, g.adjV, RV, RU.rank);
    uint32_t* tmp = r.alloc<uint32_t>(g.m);
    sort_side(r, RU, tmp);
    sort_side(r, RV, tmp);
  }
  Dev h = g;
  h.offU = RU.offN;
  h.adjU = RU.adjN;
  h.offV = RV.offN;
  h.adjV = RV.adjN;
  return h;
}

// Scratch and state of one decomposition.
struct State {
  Dev g;
  uint32_t* ld;       // live degree of v
  uint32_t* adjL;     // live (partition-ordered) copy of adjV
  uint32_t* tmp;      // compaction staging
  uint64_t* wc;       // static wedge work per u
  uint64_t* support;
  uint64_t* init;     // ⋈^init
  uint32_t* part;
  uint32_t* F;
  uint2* tier[4];     // aggregation tiers 0-2, [3] = classify's hub queue
  uint32_t* vflag;
  uint32_t* touched;
  Counters* c;
  unsigned long long* hist_w;
  uint32_t* hist_n;
  unsigned long long* sum_d2;
  uint32_t nslots;
  uint32_t *slot_cnt, *slot_touch, *slot_dup;  // FD heavy path: dense counters per CTA
  uint32_t* win_bnd;  // tier-2 window bounds, win_cap per CTA
  uint64_t win_cap;
  uint32_t win_split = 1;  // window groups per tier-2 start in the next launch
  uint32_t win_pre = 1024;
  bool prof = std::getenv("PBNG_TRACE") != nullptr;
  // chunked compaction of long lists
  uint2* comp_task;
  uint32_t *comp_tbase, *comp_oldL, *comp_cnt, *comp_ntask;
  // vertex-priority counting (Alg.1)
  bool vp;
  uint32_t* cutU;                 // static prefix of N_u ranked above u
  uint32_t* cutV;                 // live prefix of N_v ranked above v (per count)
  unsigned long long* sum_min;    // ∧_cnt = Σ_(u,v) min(d_u, d_v)
  const SideRank* RU;
  const SideRank* RV;
  uint32_t* cc = nullptr;     // k-tip level retrieval: union-find parents
  uint32_t* cut_e = nullptr;  // ... and per U-edge partner-prefix lengths
  uint32_t idspace = 0;       // 1 + largest live id (tier-2 window range; ids above are all peeled)
  // tier 1 (agg_hash.cuh): degree-mass windows, window-bound rows of long V lists
  uint32_t* wb = nullptr;
  uint32_t* rowid = nullptr;
  uint32_t* rows = nullptr;
  uint32_t cb = 0, dlim = 0;  // count-field bits of a packed slot; starts need fewer lists than dlim
  bool stats = false;         // count live-partner decrements (PBNG_OPT_STATS / _DEFER)
  // list-split mode of tier 2 (k_agg_lsplit): per-start global counters + finish tickets
  uint32_t* ls_cnt = nullptr;
  uint32_t* ls_done = nullptr;
  uint32_t ls_range = 0;      // > 0: the next PEEL launch uses list-split units over ids [0, ls_range)
};

uint32_t choose_slots(const Run& r, uint32_t nU) {
  size_t freeb = 0, totalb = 0;
  CK(cudaMemGetInfo(&freeb, &totalb));
  const size_t per = (size_t)12 * std::max<uint32_t>(nU, 1);
  size_t budget = std::min<size_t>(freeb / 3, (size_t)48 << 30);
  size_t n = budget / per;
  n = std::min<size_t>(n, (size_t)r.nsm);
  return (uint32_t)std::max<size_t>(n, 1);
}

void alloc_state(Run& r, State& S, const Dev& g, bool need_live, const SideRank& RU, const SideRank& RV, bool vp) {
  S.g = g;
  S.idspace = g.nU;
  S.vp = vp;
  S.RU = &RU;
  S.RV = &RV;
  S.ld = r.alloc<uint32_t>(g.nV);
  // g is the relabeled graph owned by this call: CD deletes from its V lists in place
  S.adjL = const_cast<uint32_t*>(g.adjV);
  S.tmp = need_live ? r.alloc<uint32_t>(g.m) : nullptr;
  if (need_live) {
    const size_t cap = 2 * (g.m / kCompChunk) + 2;
    S.comp_task = r.alloc<uint2>(cap);
    S.comp_cnt = r.alloc<uint32_t>(cap);
    S.comp_tbase = r.alloc<uint32_t>(g.nV);
    S.comp_oldL = r.alloc<uint32_t>(g.nV);
    S.comp_ntask = r.alloc<uint32_t>(1);
  }
  S.wc = r.alloc<uint64_t>(g.nU);
  S.support = r.alloc<uint64_t>(g.nU);
  S.init = need_live ? r.alloc<uint64_t>(g.nU) : nullptr;
  S.part = r.alloc<uint32_t>(g.nU);
  S.F = r.alloc<uint32_t>(g.nU);
  for (int t = 0; t < 4; t++) S.tier[t] = r.alloc<uint2>(std::max(g.nU, g.nV));
  S.vflag = r.alloc<uint32_t>(g.nV);
  S.touched = r.alloc<uint32_t>(g.nV);
  S.c = r.alloc<Counters>(1);
  S.hist_w = r.alloc<unsigned long long>(kBins);
  S.hist_n = r.alloc<uint32_t>(kBins);
  S.sum_d2 = r.alloc<unsigned long long>(2);
  S.sum_min = S.sum_d2 + 1;
  CK(cudaMemsetAsync(S.vflag, 0, (size_t)std::max<uint32_t>(g.nV, 1) * 4, r.st));
  CK(cudaMemsetAsync(S.c, 0, sizeof(Counters), r.st));
  CK(cudaMemsetAsync(S.sum_d2, 0, 16, r.st));
  r.pre(PBNG_K_INIT);
  k_init_v<<<r.nsm * 4, 256, 0, r.st>>>(g.nV, g.offV, S.ld, S.sum_d2);
  r.post(PBNG_K_INIT);
  r.pre(PBNG_K_INIT);
  k_init_u<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.offU, g.adjU, g.offV, S.wc, S.part, S.sum_min);
  r.post(PBNG_K_INIT);
  S.cutU = S.cutV = nullptr;
  if (vp) {
    S.cutU = r.alloc<uint32_t>(g.nU);
    S.cutV = r.alloc<uint32_t>(g.nV);
    r.pre(PBNG_K_COUNT_VP);
    k_vp_cut_u<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.offU, g.adjU, RV.binoff, RV.dmax, S.cutU);
    r.post(PBNG_K_COUNT_VP);
  }
  // tier 1: packed slot = (x + 1) << cb | w, x + 1 <= nU needs bitlen(nU) key bits
  const uint32_t keybits = g.nU ? 32u - (uint32_t)__builtin_clz(g.nU) : 1u;
  S.cb = 32u - keybits;
  S.dlim = S.cb >= 7 ? kHashLists : (1u << S.cb);
  S.wb = r.alloc<uint32_t>(kHW + 1);
  r.pre(PBNG_K_INIT);
  k_mass_windows<<<1, 64, 0, r.st>>>(g.nU, g.m, g.offU, S.wb);
  r.post(PBNG_K_INIT);
  S.rowid = r.alloc<uint32_t>(g.nV);
  uint32_t* nrows = r.alloc<uint32_t>(1);
  CK(cudaMemsetAsync(nrows, 0, 4, r.st));
  if (g.nV) {
    r.pre(PBNG_K_INIT);
    k_rows_ids<<<r.nsm * 8, 256, 0, r.st>>>(g.nV, g.offV, S.rowid, nrows);
    r.post(PBNG_K_INIT);
  }
  uint32_t hrows = 0;
  CK(cudaMemcpyAsync(&hrows, nrows, 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  S.rows = r.alloc<uint32_t>((size_t)hrows * (kHW + 1));
  if (hrows) {
    r.pre(PBNG_K_INIT);
    k_rows_fill<<<r.nsm * 8, 256, 0, r.st>>>(g.nV, nullptr, nullptr, S.rowid, g.offV, S.adjL, S.ld, S.wb, S.rows);
    r.post(PBNG_K_INIT);
  }
  const uint64_t wmax = ((uint64_t)std::max(g.nU, g.nV) + kWinIds - 1) / kWinIds;
  // per-CTA tables of starts with up to win_pre lists: bounds + chunk prefixes
  // ((W+1) u32 each per list) and list bases (u64); about 8 MB per CTA at most
  S.win_pre = (uint32_t)std::max<uint64_t>(kWinLists, std::min<uint64_t>(PBNG_WIN_PRE_MAX, (8ull << 20) / (8 * (wmax + 1) + 8)));
  S.win_cap = 2 * (uint64_t)S.win_pre * (wmax + 1) + 2 * (uint64_t)S.win_pre + 33 * (uint64_t)S.win_pre;
  S.win_bnd = r.alloc<uint32_t>((size_t)r.nsm * kWinCtas * S.win_cap);
}

AggArgs agg_args(const State& S, int t) {
  AggArgs a;
  a.offU = S.g.offU;
  a.adjU = S.g.adjU;
  a.offV = S.g.offV;
  a.adjV = S.adjL;
  a.ld = S.ld;
  a.part = S.part;
  a.support = S.support;
  a.list = S.tier[t];
  a.count = &S.c->ntier[t];
  a.nU = S.g.nU;
  a.ticket = &S.c->ticket[t];
  a.c = S.c;
  a.cutV = S.cutV;
  a.cutU = S.cutU;
  a.win_bnd = S.win_bnd;
  a.win_cap = S.win_cap;
  a.win_split = S.win_split;
  a.win_pre = S.win_pre;
  a.win_prof = S.prof;
  a.cc = S.cc;
  a.cut_e = S.cut_e;
  a.idspace = S.idspace;
  a.rowid = S.rowid;
  a.rows = S.rows;
  a.wb = S.wb;
  a.cb = S.cb;
  a.tier2 = S.tier[2];
  a.ntier2 = &S.c->ntier[2];
  a.stats = S.stats;
  return a;
}

template <int MODE>
void launch_agg(Run& r, State& S, const uint32_t* ntier) {
  // ntier: tier sizes read back by the host (launch only non-empty tiers)
  if (ntier[0]) {
    r.pre(PBNG_K_AGG_WARP);
    k_agg_warp<MODE><<<r.nsm * 3, kWarpTierThreads, warp_tier_smem(), r.st>>>(agg_args(S, 0));
    r.post(PBNG_K_AGG_WARP);
  }
  if (ntier[1]) {
    r.pre(PBNG_K_AGG_HASH);
    k_agg_hash<MODE><<<r.nsm * kHashCtas, kHashThreads, hash_smem(), r.st>>>(agg_args(S, 1));
    r.post(PBNG_K_AGG_HASH);
  }
  if (MODE == 1 && S.ls_range) {
    r.pre(PBNG_K_AGG_CTA);
    k_agg_lsplit<1><<<r.nsm * kWinCtas, kWinThreads, win_smem(), r.st>>>(agg_args(S, 2), S.ls_range, S.ls_cnt,
                                                                        S.ls_done);
    r.post(PBNG_K_AGG_CTA);
    S.ls_range = 0;
  } else if (ntier[2] || ntier[1]) {  // tier 1 passes on starts with a window above its capacity
    r.pre(PBNG_K_AGG_CTA);
    k_agg_win<MODE><<<r.nsm * kWinCtas, kWinThreads, win_smem(), r.st>>>(agg_args(S, 2));
    r.post(PBNG_K_AGG_CTA);
  }
}

void reset_tiers(Run& r, State& S) {
  CK(cudaMemsetAsync(&S.c->ntier[0], 0, 8 * sizeof(uint32_t), r.st));  // ntier[3] + ticket[4] + nbig
}

// Tier-2 starts are split into units (groups of coarse windows, or equal id
// ranges of at least kMinSpan ids when a start has fewer windows than the
// split wants) when a batch has fewer than two starts per SM, so that small
// batches of heavy starts still occupy every SM.  A unit should carry about
// kMinUnitWedges wedges or more (wedges = the batch's classified wedges).
#ifndef PBNG_LSPLIT
#define PBNG_LSPLIT 1
#endif
#ifndef PBNG_MIN_SPAN
#define PBNG_MIN_SPAN 2048
#endif
constexpr uint64_t kMinSpan = PBNG_MIN_SPAN;
constexpr uint64_t kMinUnitWedges = 1u << 16;
uint32_t pick_split(const Run& r, uint32_t n2, uint32_t idspace, uint64_t wedges = ~0ull) {
  if (n2 == 0 || idspace <= kMinSpan) return 1;
  const uint64_t want = (2ull * (uint64_t)r.nsm * kWinCtas + n2 - 1) / n2;
  const uint64_t by_ids = ((uint64_t)idspace + kMinSpan - 1) / kMinSpan;
  const uint64_t by_work = std::max<uint64_t>(1, wedges / n2 / kMinUnitWedges);
  return (uint32_t)std::max<uint64_t>(1, std::min({want, by_ids, by_work}));
}

// List-split mode (k_agg_lsplit) for a small tier-2 batch over a small live id range.
constexpr uint64_t kLsCap = 1ull << 24;  // global counters (64 MB)
#ifndef PBNG_LS_MAX_IDS
#define PBNG_LS_MAX_IDS 8192
#endif
// live id ranges up to this use list-split units (measured on config 5: at 12K-28K live
// ids the windowed kernel split by id range is faster; at a few thousand and below,
// list-split units are)
constexpr uint32_t kLsMaxIds = PBNG_LS_MAX_IDS < kWinBitWords ? PBNG_LS_MAX_IDS : kWinBitWords;
void plan_lsplit(Run& r, State& S, const Counters& hc) {
  S.ls_range = 0;
  const uint64_t n2 = (uint64_t)hc.ntier[2] + hc.ntier[1];  // tier 1 may pass starts on
  const uint64_t stride = ((uint64_t)S.idspace + 3) & ~3ull;
  if (hc.ntier[2] == 0 || hc.ntier[2] >= 2u * (uint32_t)r.nsm * kWinCtas || S.idspace > kLsMaxIds ||
      n2 * stride > kLsCap)
    return;
  if (!S.ls_cnt) {
    S.ls_cnt = r.alloc<uint32_t>(kLsCap);
    S.ls_done = r.alloc<uint32_t>(kLsCap / 4);
  }
  CK(cudaMemsetAsync(S.ls_cnt, 0, n2 * stride * 4, r.st));
  CK(cudaMemsetAsync(S.ls_done, 0, n2 * 4, r.st));
  S.ls_range = S.idspace;
  const uint64_t want = (2ull * (uint64_t)r.nsm * kWinCtas + hc.ntier[2] - 1) / hc.ntier[2];
  const uint64_t by_work = std::max<uint64_t>(1, hc.wedges / hc.ntier[2] / kMinUnitWedges);
  S.win_split = (uint32_t)std::max<uint64_t>(1, std::min(want, by_work));
}


// Vertex-priority count (Alg.1, kernels_vp.cuh) of every unassigned u on the
// live graph: starts in U, then starts in V; supports accumulate atomically.
void vp_count_live(Run& r, State& S) {
  const Dev& g = S.g;
  CK(cudaMemsetAsync(S.support, 0, (size_t)g.nU * 8, r.st));
  r.pre(PBNG_K_COUNT_VP);
  k_vp_cut_v<<<r.nsm * 8, 256, 0, r.st>>>(g.nV, g.offV, S.adjL, S.ld, S.RU->binoff, S.RU->dmax, S.cutV);
  r.post(PBNG_K_COUNT_VP);
  // starts in U
  reset_tiers(r, S);
  r.pre(PBNG_K_CLASSIFY);
  k_vp_classify<0><<<r.nsm * 8, 256, 0, r.st>>>(g.nU, agg_args(S, 0), S.tier[0], S.tier[1], S.tier[2], S.tier[3],
                                                 kHashMaxPb, S.dlim);
  r.post(PBNG_K_CLASSIFY);
  r.pre(PBNG_K_CLASSIFY);
  k_vp_classify_big<0><<<r.nsm * 2, 512, 0, r.st>>>(agg_args(S, 0), S.tier[3], S.tier[0], S.tier[1], S.tier[2],
                                                    kHashMaxPb, S.dlim);
  r.post(PBNG_K_CLASSIFY);
  S.win_split = pick_split(r, r.readback(S.c).ntier[2], g.nU);
  r.pre(PBNG_K_AGG_WARP);
  k_vp_agg_warp<0><<<r.nsm * 3, kWarpTierThreads, warp_tier_smem(), r.st>>>(agg_args(S, 0));
  r.post(PBNG_K_AGG_WARP);
  r.pre(PBNG_K_AGG_HASH);
  k_vp_agg_hash<<<r.nsm * kHashCtas, kHashThreads, hash_smem(), r.st>>>(agg_args(S, 1));
  r.post(PBNG_K_AGG_HASH);
  r.pre(PBNG_K_AGG_CTA);
  k_vp_agg_win<0><<<r.nsm * kWinCtas, kWinThreads, win_smem(), r.st>>>(agg_args(S, 2));
  r.post(PBNG_K_AGG_CTA);
  // starts in V
  reset_tiers(r, S);
  r.pre(PBNG_K_CLASSIFY);
  k_vp_classify<1><<<r.nsm * 8, 256, 0, r.st>>>(g.nV, agg_args(S, 0), S.tier[0], S.tier[1], S.tier[2], S.tier[3],
                                                 kCtaCap, 0xFFFFFFFFu);
  r.post(PBNG_K_CLASSIFY);
  r.pre(PBNG_K_CLASSIFY);
  k_vp_classify_big<1><<<r.nsm * 2, 512, 0, r.st>>>(agg_args(S, 0), S.tier[3], S.tier[0], S.tier[1], S.tier[2],
                                                    kCtaCap, 0xFFFFFFFFu);
  r.post(PBNG_K_CLASSIFY);
  S.win_split = pick_split(r, r.readback(S.c).ntier[2], g.nV);
  r.pre(PBNG_K_AGG_WARP);
  k_vp_agg_warp<1><<<r.nsm * 3, kWarpTierThreads, warp_tier_smem(), r.st>>>(agg_args(S, 0));
  r.post(PBNG_K_AGG_WARP);
  r.pre(PBNG_K_AGG_CTA);
  k_vp_agg_mid<1><<<r.nsm * kMidCtas, kMidThreads, mid_smem(), r.st>>>(agg_args(S, 1));
  r.post(PBNG_K_AGG_CTA);
  r.pre(PBNG_K_AGG_CTA);
  k_vp_agg_win<1><<<r.nsm * kWinCtas, kWinThreads, win_smem(), r.st>>>(agg_args(S, 2));
  r.post(PBNG_K_AGG_CTA);
}

// Butterfly count of every unassigned u (initial count, and §5.1 re-count).
void count_live(Run& r, State& S) {
  if (S.vp) {
    vp_count_live(r, S);
    return;
  }
  CK(cudaMemsetAsync(S.support, 0, (size_t)S.g.nU * 8, r.st));  // tier 2 accumulates
  reset_tiers(r, S);
  r.pre(PBNG_K_CLASSIFY);
  k_classify<0><<<r.nsm * 8, 256, 0, r.st>>>(S.g.nU, nullptr, nullptr, S.g.offU, S.g.adjU, S.ld, S.part,
                                               S.support, S.tier[0], S.tier[1], S.tier[2], S.tier[3], nullptr, 0,
                                               S.c, kHashMaxPb, S.dlim);
  r.post(PBNG_K_CLASSIFY);
  r.pre(PBNG_K_CLASSIFY);
  k_classify_big<0><<<r.nsm * 2, 512, 0, r.st>>>(S.tier[3], S.c, S.g.offU, S.g.adjU, S.ld, S.support, S.tier[0],
                                                  S.tier[1], S.tier[2], nullptr, 0, S.c, kHashMaxPb, S.dlim);
  r.post(PBNG_K_CLASSIFY);
  const Counters hc = r.readback(S.c);
  S.win_split = pick_split(r, hc.ntier[2], S.idspace);
  launch_agg<0>(r, S, hc.ntier);
}

// live entries: part[x] > thr (default: not yet peeled; PBNG- replay: partitions above thr)
void compact(Run& r, State& S, uint32_t epoch, bool force = false, uint32_t thr = kUnassigned - 1) {
  (void)epoch;
  const uint32_t big = kCompChunk;
  CK(cudaMemsetAsync(&S.c->ntouched, 0, 4, r.st));
  CK(cudaMemsetAsync(S.comp_ntask, 0, 4, r.st));
  r.pre(PBNG_K_COMPACT);
  k_collect_touched<<<r.nsm * 8, 256, 0, r.st>>>(S.g.nV, S.vflag, S.ld, big, force, S.touched, S.c);
  r.post(PBNG_K_COMPACT);
  r.pre(PBNG_K_COMPACT);
  k_compact<<<r.nsm * 8, 256, 0, r.st>>>(S.touched, &S.c->ntouched, S.g.offV, S.adjL, S.tmp, S.ld, S.part, big,
                                         S.c, thr);
  r.post(PBNG_K_COMPACT);
  // lists of >= big entries: chunked over CTAs
  r.pre(PBNG_K_COMPACT);
  k_compact_plan<<<r.nsm * 2, 256, 0, r.st>>>(S.touched, &S.c->ntouched, S.ld, big, S.comp_task, S.comp_tbase,
                                              S.comp_oldL, S.comp_ntask);
  r.post(PBNG_K_COMPACT);
  r.pre(PBNG_K_COMPACT);
  k_compact_count<<<r.nsm * 4, kCompThreads, 0, r.st>>>(S.comp_task, S.comp_ntask, S.touched, S.comp_oldL, S.g.offV,
                                                        S.adjL, S.tmp, S.part, S.comp_cnt, thr);
  r.post(PBNG_K_COMPACT);
  r.pre(PBNG_K_COMPACT);
  k_compact_scan<<<r.nsm, 256, 0, r.st>>>(S.touched, &S.c->ntouched, big, S.comp_tbase, S.comp_oldL, S.comp_cnt,
                                          S.ld, S.c);
  r.post(PBNG_K_COMPACT);
  r.pre(PBNG_K_COMPACT);
  k_compact_scatter<<<r.nsm * 4, kCompThreads, 0, r.st>>>(S.comp_task, S.comp_ntask, S.touched, S.comp_oldL,
                                                          S.comp_tbase, S.comp_cnt, S.g.offV, S.ld, S.adjL, S.tmp,
                                                          S.part, thr);
  r.post(PBNG_K_COMPACT);
  // window-bound rows of the compacted lists (tier 1)
  r.pre(PBNG_K_COMPACT);
  k_rows_fill<<<r.nsm * 8, 256, 0, r.st>>>(0, S.touched, &S.c->ntouched, S.rowid, S.g.offV, S.adjL, S.ld, S.wb,
                                           S.rows);
  r.post(PBNG_K_COMPACT);
}

struct Plan {
  std::vector<uint64_t> bounds;  // bounds[0] = 0 ... bounds[nparts] = inf
  uint32_t nparts = 0;
};

// Coarse-grained decomposition (Alg.4 structure P:799-816, tip P:982-991).
struct TraceRow {
  uint32_t pid, nF, t0, t1, t2;
  unsigned long long wedges, w2cum;  // batch wedges; cumulative tier-2 wedges after classify
  bool recount;
  uint32_t idspace, split;
  cudaEvent_t a, m, b;
};

void run_cd(Run& r, State& S, uint32_t P, uint32_t opts, Plan& plan, pbng_stats& st) {
  // PBNG_TRACE=1: one stderr line per CD iteration (development aid)
  const bool trace = std::getenv("PBNG_TRACE") != nullptr;
  std::vector<TraceRow> rows;
  const bool del = !(opts & PBNG_OPT_NO_DELETE);
  const uint32_t nU = S.g.nU;
  std::vector<unsigned long long> hw(kBins);
  std::vector<uint32_t> hn(kBins);
  unsigned long long sums[2] = {0, 0};  // Σ_v d_v^2, Σ_(u,v) min(d_u, d_v)
  CK(cudaMemcpyAsync(sums, S.sum_d2, 16, cudaMemcpyDeviceToHost, r.st));
  plan.bounds.assign(1, 0);
  double scale = 1.0;  // two-way adaptive target, second adaptation
  uint32_t epoch = 0;
  for (uint32_t pid = 0; pid < P; pid++) {
    // --- partition start: ⋈^init snapshot + weighted support histogram
    CK(cudaMemsetAsync(S.hist_w, 0, kBins * 8, r.st));
    CK(cudaMemsetAsync(S.hist_n, 0, kBins * 4, r.st));
    CK(cudaMemsetAsync(&S.c->live_wc, 0, 24, r.st));
    r.pre(PBNG_K_RANGE);
    k_range_hist<<<r.nsm, 1024, hist_smem(), r.st>>>(nU, S.part, S.support, S.wc, S.init, S.hist_w, S.hist_n,
                                                     S.c);
    r.post(PBNG_K_RANGE);
    CK(cudaMemcpyAsync(hw.data(), S.hist_w, kBins * 8, cudaMemcpyDeviceToHost, r.st));
    CK(cudaMemcpyAsync(hn.data(), S.hist_n, kBins * 4, cudaMemcpyDeviceToHost, r.st));
    const Counters hc0 = r.readback(S.c);
    if (hc0.live_n == 0) break;
#ifndef PBNG_LIVE_IDSPACE
#define PBNG_LIVE_IDSPACE 1
#endif
    // the live set only shrinks inside a partition: partners above the
    // largest live id are all peeled, so tier-2 windows stop there
    if (PBNG_LIVE_IDSPACE) S.idspace = (uint32_t)hc0.max_live;
    // --- find_range: smallest bin whose cumulative work reaches tgt
    uint64_t bound = kInf;
    if (pid + 1 < P) {
      double tgt = scale * (double)hc0.live_wc / (double)(P - pid);  // first adaptation
      tgt = std::max(tgt, 1.0);
      uint32_t b0 = 0;
      while (b0 < kBins && hn[b0] == 0) b0++;
      unsigned long long cum = 0;
      uint32_t b = 0;
      for (; b < kBins; b++) {
        cum += hw[b];
        if ((double)cum >= tgt) break;
      }
      b = std::max(b, b0);
      bound = (b + 1 < kBins) ? key_lo(b + 1) : kInf;
    }
    plan.bounds.push_back(bound);
    // --- peel batches until no live support is below the bound
    unsigned long long first_wc = 0, part_wc = 0;
    bool first = true;
    if (!del) {
      epoch++;
      CK(cudaMemsetAsync(&S.c->ntouched, 0, 4, r.st));
    }
    for (;;) {
      CK(cudaMemsetAsync(S.c, 0, offsetof(Counters, ntouched), r.st));
      if (del) {
        epoch++;
        CK(cudaMemsetAsync(&S.c->ntouched, 0, 4, r.st));
      }
      r.pre(PBNG_K_SELECT);
      k_select<<<r.nsm * 8, 256, 0, r.st>>>(nU, S.part, S.support, S.wc, bound, pid, S.F, S.c);
      r.post(PBNG_K_SELECT);
      r.pre(PBNG_K_CLASSIFY);
      k_classify<1><<<r.nsm * 8, 256, 0, r.st>>>(nU, S.F, &S.c->nF, S.g.offU, S.g.adjU, S.ld, S.part, S.support,
                                                   S.tier[0], S.tier[1], S.tier[2], S.tier[3], S.vflag, epoch,
                                                   S.c, kHashMaxPb, S.dlim);
      r.post(PBNG_K_CLASSIFY);
      r.pre(PBNG_K_CLASSIFY);
      k_classify_big<1><<<r.nsm * 2, 512, 0, r.st>>>(S.tier[3], S.c, S.g.offU, S.g.adjU, S.ld, S.support,
                                                      S.tier[0], S.tier[1], S.tier[2], S.vflag, epoch, S.c,
                                                      kHashMaxPb, S.dlim);
      r.post(PBNG_K_CLASSIFY);
      const Counters hc = r.readback(S.c);
      if (hc.nF == 0) break;
      st.rho_cd_iters++;
      if (first) first_wc = hc.sel_wc;
      first = false;
      part_wc += hc.sel_wc;
      if (bound == kInf) {
        // every live vertex is in this batch: nobody is left to update
        if (del) compact(r, S, epoch);
        continue;
      }
      // re-count cost (g10): ∧_cnt = Σ min(d_u, d_v) for vertex-priority
      // counting; the one-sided count costs Σ_v ld_v^2
      const unsigned long long recount_cost = S.vp ? sums[1] : sums[0] - hc.ld2_drop;
      const bool recount = !(opts & PBNG_OPT_NO_RECOUNT) &&
                           ((opts & PBNG_OPT_FORCE_RECOUNT) || hc.wedges > recount_cost);
      cudaEvent_t ta = trace ? r.event() : nullptr, tm = nullptr;
      if (recount) {
        // §5.1: re-compute supports of all remaining vertices
        if (del) compact(r, S, epoch);
        count_live(r, S);
        st.recounts++;
      } else {
        S.win_split = pick_split(r, hc.ntier[2], S.idspace, hc.wedges);
        if (PBNG_LSPLIT) plan_lsplit(r, S, hc);
        launch_agg<1>(r, S, hc.ntier);
        if (trace) tm = r.event();
        if (del) compact(r, S, epoch);
      }
      if (trace) {
        TraceRow row{pid, hc.nF, hc.ntier[0], hc.ntier[1], hc.ntier[2], hc.wedges, hc.tier_wedges[2], recount,
                     S.idspace, S.win_split, ta, tm ? tm : ta, r.event()};
        rows.push_back(row);
      }
    }
    if (del) compact(r, S, epoch, true);  // partition end: every list grouped by partition for FD
    scale = part_wc ? (double)first_wc / (double)part_wc : 1.0;
  }
  plan.nparts = (uint32_t)plan.bounds.size() - 1;
  if (!del) {
    // PBNG- (no dynamic graph updates): the lists kept every peeled
    // entry during CD; FD's induced-subgraph layout (each N_v grouped by
    // partition, latest first) is built once now, by replaying the partition-end
    // compaction per partition: step p moves the entries of partition p behind
    // the entries of later partitions.
    for (uint32_t p = 0; p < plan.nparts; p++) {
      CK(cudaMemsetAsync(S.vflag, 1, (size_t)S.g.nV * 4, r.st));
      compact(r, S, epoch, true, p);
    }
  }
  if (plan.nparts) plan.bounds.back() = kInf;
  if (trace) {
    const Counters hc = r.readback(S.c);
    std::fprintf(stderr, "tier2 cycles: tabled_starts=%llu precompute=%llu bitmap=%llu dense=%llu | untabled=%llu "
                 "n_untabled=%llu n_tabled=%llu | windows=%llu over=%llu dense_passes=%llu\n", hc.prof[0], hc.prof[1],
                 hc.prof[2], hc.prof[3], hc.prof2[0], hc.prof2[1], hc.prof2[2], hc.dbg[0], hc.dbg[1], hc.dbg[2]);
    std::fprintf(stderr, "tier2 dense: subtab=%llu mark=%llu sweep=%llu | entries=%llu windows=%llu lists_per_batch_sum=%llu "
                 "| mark_setup=%llu mark_loop=%llu\n", hc.prof3[0], hc.prof3[1], hc.prof3[2], hc.prof3[3], hc.prof3[4],
                 hc.prof3[5], hc.prof3[6], hc.prof3[7]);
    for (const TraceRow& t : rows)
      std::fprintf(stderr, "cd pid=%u nF=%u tiers=%u/%u/%u wedges=%llu w2cum=%llu recount=%d ms=%.3f agg_ms=%.3f "
                   "idspace=%u split=%u\n", t.pid, t.nF, t.t0, t.t1, t.t2, t.wedges, t.w2cum, (int)t.recount,
                   elapsed(t.a, t.b), elapsed(t.a, t.m), t.idspace, t.split);
  }
}

// Fine-grained decomposition -> theta.
// FD of heavy small partitions on the whole GPU, host-driven rounds (kernels_fd.cuh).
void fd_grid(Run& r, State& S, const std::vector<uint32_t>& heavy, const std::vector<uint32_t>& hoff,
             const std::vector<uint32_t>& hcount, const uint32_t* members, const uint64_t* seg, uint32_t* fstate,
             uint64_t* theta, unsigned long long* fdc) {
  uint32_t* lpos = r.alloc<uint32_t>(S.g.nU);
  uint32_t* sel = r.alloc<uint32_t>(1024);
  uint64_t* selpre = r.alloc<uint64_t>(1025);
  uint32_t* gcnt = r.alloc<uint32_t>(kGridCnt);
  unsigned long long* ctl = r.alloc<unsigned long long>(3);
  CK(cudaMemsetAsync(lpos, 0xFF, (size_t)S.g.nU * 4, r.st));
  CK(cudaMemsetAsync(gcnt, 0, (size_t)kGridCnt * 4, r.st));
  const bool trace = std::getenv("PBNG_TRACE") != nullptr;
  for (uint32_t p : heavy) {
    cudaEvent_t ta = trace ? r.event() : nullptr;
    uint32_t rounds = 0;
    unsigned long long edges = 0;
    const uint32_t n = hcount[p];
    const uint32_t* mem = members + hoff[p];
    const uint32_t maxsel = std::min<uint32_t>(1024, kGridCnt / n);
    r.pre(PBNG_K_FD);
    k_fdg_pos<<<(n + 255) / 256, 256, 0, r.st>>>(mem, n, lpos);
    r.post(PBNG_K_FD);
    CK(cudaMemsetAsync(ctl, 0, 24, r.st));
    for (;;) {
      r.pre(PBNG_K_FD);
      k_fdg_select<<<1, 1024, 0, r.st>>>(mem, n, S.g.offU, S.support, fstate, theta, maxsel, sel, selpre, ctl);
      r.post(PBNG_K_FD);
      unsigned long long hc[3];
      CK(cudaMemcpyAsync(hc, ctl, 24, cudaMemcpyDeviceToHost, r.st));
      CK(cudaStreamSynchronize(r.st));
      const uint32_t ns = (uint32_t)hc[1];
      if (ns == 0) break;
      rounds++;
      edges += hc[2];
      const uint32_t nc = ns * n;
      r.pre(PBNG_K_FD);
      k_fdg_agg<<<r.nsm * 2, kGridThreads, (size_t)nc * 4, r.st>>>(sel, selpre, ns, n, S.g.offU, S.g.adjU, S.g.offV,
                                                                 seg, S.adjL, lpos, fstate, gcnt, fdc);
      r.post(PBNG_K_FD);
      r.pre(PBNG_K_FD);
      k_fdg_apply<<<std::max<uint32_t>(1, std::min<uint32_t>((nc + 255) / 256, r.nsm * 4)), 256, 0, r.st>>>(
          nc, n, mem, gcnt, S.support, fdc + 1);
      r.post(PBNG_K_FD);
    }
    if (trace) {
      cudaEvent_t tb = r.event();
      CK(cudaEventSynchronize(tb));
      std::fprintf(stderr, "fd-grid part=%u members=%u rounds=%u edges=%llu ms=%.3f\n", p, n, rounds, edges,
                   elapsed(ta, tb));
    }
  }
}

void run_fd(Run& r, State& S, const Plan& plan, uint64_t* theta, pbng_stats& st, float& ms_build, uint32_t opts) {
  const uint32_t np = plan.nparts, nU = S.g.nU;
  cudaEvent_t e0 = r.event();
  uint32_t* pcount = r.alloc<uint32_t>(2 * np);  // [0, np) FD members, [np, 2np) all vertices
  uint32_t* poff = r.alloc<uint32_t>(np + 1);
  uint32_t* pcur = r.alloc<uint32_t>(np);
  unsigned long long* work = r.alloc<unsigned long long>(np);
  uint32_t* order = r.alloc<uint32_t>(np);
  uint32_t* members = r.alloc<uint32_t>(nU);
  uint32_t* sel = r.alloc<uint32_t>(nU);
  uint32_t* selpb = r.alloc<uint32_t>(nU);
  uint32_t* fstate = r.alloc<uint32_t>(nU);
  uint32_t* cand = r.alloc<uint32_t>(nU);
  uint32_t* cand2 = r.alloc<uint32_t>(nU);
  uint32_t* sel2 = r.alloc<uint32_t>(nU);
  uint32_t* bigl = r.alloc<uint32_t>(nU);
  uint64_t* seg = r.alloc<uint64_t>(S.g.m);
  unsigned long long* fdc = r.alloc<unsigned long long>(3);  // wedges, updates, steps
  uint32_t* misc = r.alloc<uint32_t>(3);                     // ticket, rounds_max, heavy count
  CK(cudaMemsetAsync(pcount, 0, (size_t)np * 8, r.st));
  CK(cudaMemsetAsync(pcur, 0, (size_t)np * 4, r.st));
  CK(cudaMemsetAsync(work, 0, (size_t)np * 8, r.st));
  CK(cudaMemsetAsync(fstate, 0, (size_t)nU * 4, r.st));
  CK(cudaMemsetAsync(fdc, 0, 24, r.st));
  CK(cudaMemsetAsync(misc, 0, 12, r.st));
  r.pre(PBNG_K_FD_BUILD);
  k_part_count<<<r.nsm * 4, 256, np * 8, r.st>>>(nU, S.part, S.init, np, pcount, pcount + np);
  r.post(PBNG_K_FD_BUILD);
  std::vector<uint32_t> hcount(np), hoff(np + 1);
  CK(cudaMemcpyAsync(hcount.data(), pcount, (size_t)np * 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  hoff[0] = 0;
  for (uint32_t i = 0; i < np; i++) hoff[i + 1] = hoff[i] + hcount[i];
  CK(cudaMemcpyAsync(poff, hoff.data(), (size_t)(np + 1) * 4, cudaMemcpyHostToDevice, r.st));
  r.pre(PBNG_K_FD_BUILD);
  k_part_scatter<<<r.nsm * 8, 256, 0, r.st>>>(nU, S.part, S.init, poff, pcur, members, fstate, theta);
  r.post(PBNG_K_FD_BUILD);
  r.pre(PBNG_K_FD_BUILD);
  k_fd_seg<<<r.nsm * 8, 256, np * 8, r.st>>>(nU, S.g.offU, S.g.adjU, S.g.offV, S.adjL, S.part, np, seg, work,
                                              misc + 2);
  r.post(PBNG_K_FD_BUILD);
  std::vector<unsigned long long> hwork(np);
  uint32_t hheavy = 0;
  CK(cudaMemcpyAsync(hwork.data(), work, (size_t)np * 8, cudaMemcpyDeviceToHost, r.st));
  CK(cudaMemcpyAsync(&hheavy, misc + 2, 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  // dense-counter slots only when some FD vertex outgrows the CTA table
  S.nslots = hheavy ? choose_slots(r, nU) : (uint32_t)r.nsm;
  const size_t slot_elems = hheavy ? (size_t)S.nslots * nU : 1;
  S.slot_cnt = r.alloc<uint32_t>(slot_elems);
  S.slot_touch = r.alloc<uint32_t>(slot_elems);
  S.slot_dup = r.alloc<uint32_t>(slot_elems);
  CK(cudaMemsetAsync(S.slot_cnt, 0, slot_elems * 4, r.st));
  // workload-aware scheduling: LPT order
  std::vector<uint32_t> all(np), ord, heavy;
  for (uint32_t i = 0; i < np; i++) all[i] = i;
  std::stable_sort(all.begin(), all.end(), [&](uint32_t a, uint32_t b) { return hwork[a] > hwork[b]; });
  // heavy small partitions (work far above the per-SM average, few members) go to the grid path
  unsigned long long wsum = 0;
  for (uint32_t i = 0; i < np; i++) wsum += hwork[i];
  const bool force_grid = (opts & PBNG_OPT_FD_GRID) != 0;
  for (uint32_t p : all) {
    const bool small = hcount[p] >= 1 && hcount[p] <= kGridMaxMembers;
    if (small && (force_grid || (double)hwork[p] > 4.0 * (double)wsum / (double)r.nsm)) heavy.push_back(p);
    else ord.push_back(p);
  }
  if (!ord.empty())
    CK(cudaMemcpyAsync(order, ord.data(), (size_t)ord.size() * 4, cudaMemcpyHostToDevice, r.st));
  CK(cudaMemcpyAsync(S.support, S.init, (size_t)nU * 8, cudaMemcpyDeviceToDevice, r.st));
  cudaEvent_t e1 = r.event();
  FdArgs a;
  a.nU = nU;
  a.offU = S.g.offU;
  a.adjU = S.g.adjU;
  a.offV = S.g.offV;
  a.adjL = S.adjL;
  a.seg = seg;
  a.poff = poff;
  a.pall = pcount + np;
  a.order = order;
  a.nparts = (uint32_t)ord.size();
  a.ticket = misc;
  a.members = members;
  a.sel = sel;
  a.selpb = selpb;
  a.s = S.support;
  a.state = fstate;
  a.cand = cand;
  a.cand2 = cand2;
  a.sel2 = sel2;
  a.bigl = bigl;
  a.theta = theta;
  a.slot_cnt = S.slot_cnt;
  a.slot_touch = S.slot_touch;
  a.slot_dup = S.slot_dup;
  a.wedges = fdc;
  a.updates = fdc + 1;
  a.rounds_max = misc + 1;
  const bool trace = std::getenv("PBNG_TRACE") != nullptr;
  a.ptrace = nullptr;
  if (trace) {
    a.ptrace = r.alloc<unsigned long long>((size_t)8 * np);
    CK(cudaMemsetAsync(a.ptrace, 0, (size_t)64 * np, r.st));
  }
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>({np, (uint32_t)r.nsm, S.nslots}));
  if (a.nparts) {
    r.pre(PBNG_K_FD);
    k_fd<<<grid, kFdThreads, fd_smem(), r.st>>>(a);
    r.post(PBNG_K_FD);
  }
  if (!heavy.empty()) fd_grid(r, S, heavy, hoff, hcount, members, seg, fstate, theta, fdc);
  cudaEvent_t e2 = r.event();
  unsigned long long hf[3];
  uint32_t hm[2];
  CK(cudaMemcpyAsync(hf, fdc, 24, cudaMemcpyDeviceToHost, r.st));
  CK(cudaMemcpyAsync(hm, misc, 8, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  st.wedges_fd = hf[0];
  st.support_updates += hf[1];
  st.uv_steps += hf[2];
  st.uv_steps_fd = hf[2];
  st.updates_fd = hf[1];
  st.fd_rounds_max = hm[1];
  if (trace) {
    std::vector<unsigned long long> pt((size_t)8 * np);
    CK(cudaMemcpy(pt.data(), a.ptrace, pt.size() * 8, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < np; i++)
      std::fprintf(stderr, "fd part=%u members=%llu rounds=%llu cycles=%llu work=%llu sel=%llu bounds=%llu "
                   "light=%llu heavy=%llu\n", i, pt[8 * i + 3], pt[8 * i + 0], pt[8 * i + 1], hwork[i],
                   pt[8 * i + 4], pt[8 * i + 5], pt[8 * i + 6], pt[8 * i + 7]);
  }
  ms_build = elapsed(e0, e1);
  st.ms_fd = elapsed(e1, e2);
}

bool orient(pbng_csr U, pbng_csr V, int side, Dev& g) {
  if (side != 0 && side != 1) fail(PBNG_ERR_ARG, "side must be 0 (U) or 1 (V)");
  if (U.m != V.m) fail(PBNG_ERR_ARG, "U.m != V.m");
  if (side == 1) std::swap(U, V);
  if (U.n == 0xFFFFFFFFu || V.n == 0xFFFFFFFFu) fail(PBNG_ERR_ARG, "vertex count must be < 2^32 - 1");
  if (!U.offsets || !V.offsets || (U.m && (!U.indices || !V.indices)))
    fail(PBNG_ERR_ARG, "null CSR pointer");
  g.nU = U.n;
  g.nV = V.n;
  g.m = U.m;
  g.offU = U.offsets;
  g.adjU = U.indices;
  g.offV = V.offsets;
  g.adjV = V.indices;
  return true;
}

struct Out {
  uint64_t* tip = nullptr;
  uint32_t* part = nullptr;
  uint64_t* init = nullptr;
  uint64_t* bounds = nullptr;
  uint32_t* nparts = nullptr;
};

void decompose(const Dev& g, uint32_t P, uint32_t opts, const Out& out, pbng_stats* stats, cudaStream_t s) {
  if (P < 1 || P > PBNG_MAX_P) fail(PBNG_ERR_ARG, "P must be in [1, PBNG_MAX_P]");
  pbng_stats st;
  std::memset(&st, 0, sizeof(st));
  Run r(s);
  r.timing = (opts & (PBNG_OPT_STATS | PBNG_OPT_STATS_DEFER)) != 0;
  r.defer = (opts & PBNG_OPT_STATS_DEFER) != 0;
  if (r.defer) {  // a new deferred call replaces the previous one's spans
    for (const DeferredSpan& sp : deferred_spans()) {
      event_pool().push_back(sp.a);
      event_pool().push_back(sp.b);
    }
    deferred_spans().clear();
  }
  if (opts & PBNG_OPT_VALIDATE) validate(r, g);
  if (g.nU == 0) {
    if (out.bounds) {
      out.bounds[0] = 0;
      for (uint32_t i = 1; i <= P; i++) out.bounds[i] = kInf;
    }
    if (out.nparts) *out.nparts = 0;
    if (stats) *stats = st;
    return;
  }
  State S;
  S.stats = r.timing;
  cudaEvent_t t0 = r.event();
  SideRank RU, RV;
  const Dev gr = relabel(r, g, RU, RV);
  alloc_state(r, S, gr, true, RU, RV, !(opts & PBNG_OPT_ONESIDED_COUNT));
  count_live(r, S);
  cudaEvent_t t1 = r.event();
  const Counters c0 = r.readback(S.c);
  st.wedges_count = c0.cum_wedges;
  Plan plan;
  run_cd(r, S, P, opts, plan, st);
  cudaEvent_t t2 = r.event();
  st.partitions_used = plan.nparts;
  const Counters c1 = r.readback(S.c);
  st.support_updates += c1.updates;
  st.impl[3] = c1.updates_live;
  st.wedges_cd = c1.cum_wedges - c0.cum_wedges;
  for (int i = 0; i < 3; i++) st.impl[i] = c1.dbg[i];
  for (int i = 0; i < 4; i++) st.impl_hash[i] = c1.hashc[i];
  st.uv_steps += c1.cum_steps;
  st.ms_count = elapsed(t0, t1);
  st.ms_cd = elapsed(t1, t2);
  if (out.part) {
    r.pre(PBNG_K_INIT);
    k_gather<uint32_t><<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, S.part, out.part);
    r.post(PBNG_K_INIT);
    r.pre(PBNG_K_INIT);
    k_gather<uint64_t><<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, S.init, out.init);
    r.post(PBNG_K_INIT);
    for (uint32_t i = 0; i <= P; i++) out.bounds[i] = i < plan.bounds.size() ? plan.bounds[i] : kInf;
    *out.nparts = plan.nparts;
    CK(cudaStreamSynchronize(r.st));
  }
  if (out.tip) {
    float ms_build = 0;
    uint64_t* theta = r.alloc<uint64_t>(g.nU);
    run_fd(r, S, plan, theta, st, ms_build, opts);
    st.ms_fd_build = ms_build;
    r.pre(PBNG_K_INIT);
    k_gather<uint64_t><<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, theta, out.tip);
    r.post(PBNG_K_INIT);
  }
  CK(cudaStreamSynchronize(r.st));
  st.launches = r.launches;
  if (r.timing && !r.defer) r.kernel_ms(st.ms_kernel);
  if (stats) *stats = st;
}

// One level of the k-tip hierarchy from the tip numbers: members
// U_k = {θ >= k}; non-members are deleted from the V lists (the deletion pass
// of CD), then every member aggregates its wedges inside the
// level (one-sided tiers, LINK mode) and unions with each member partner it
// shares a butterfly with; each pair is walked once, from its larger internal
// id (partner lists cut at the start, k_level_cut).  Returns the number of k-tips.
uint32_t tip_level(const Dev& g, const uint64_t* tip, uint64_t k, uint32_t* out_comp, cudaStream_t s) {
  Run r(s);
  State S;
  SideRank RU, RV;
  const Dev gr = relabel(r, g, RU, RV);
  alloc_state(r, S, gr, true, RU, RV, false);
  S.cc = r.alloc<uint32_t>(g.nU);
  uint32_t* minlab = r.alloc<uint32_t>(g.nU);
  uint32_t* dn = r.alloc<uint32_t>(1);
  CK(cudaMemsetAsync(dn, 0, 4, r.st));
  r.pre(PBNG_K_INIT);
  k_level_mark<<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, tip, k, S.part, S.cc, minlab);
  r.post(PBNG_K_INIT);
  if (g.nV) {
    CK(cudaMemsetAsync(S.vflag, 1, (size_t)g.nV * 4, r.st));  // every list may hold non-members
    compact(r, S, 0, true);
  }
  S.cut_e = r.alloc<uint32_t>(std::max<uint64_t>(gr.m, 1));
  if (gr.m) {
    r.pre(PBNG_K_INIT);
    k_level_cut<<<r.nsm * 8, 256, 0, r.st>>>(gr.nU, gr.m, gr.offU, gr.adjU, gr.offV, S.adjL, S.ld, S.part, S.cut_e);
    r.post(PBNG_K_INIT);
  }
  reset_tiers(r, S);
  r.pre(PBNG_K_CLASSIFY);
  k_classify<0><<<r.nsm * 8, 256, 0, r.st>>>(gr.nU, nullptr, nullptr, gr.offU, gr.adjU, S.ld, S.part, S.support,
                                               S.tier[0], S.tier[1], S.tier[2], S.tier[3], nullptr, 0, S.c,
                                               kHashMaxPb, S.dlim);
  r.post(PBNG_K_CLASSIFY);
  r.pre(PBNG_K_CLASSIFY);
  k_classify_big<0><<<r.nsm * 2, 512, 0, r.st>>>(S.tier[3], S.c, gr.offU, gr.adjU, S.ld, S.support, S.tier[0],
                                                  S.tier[1], S.tier[2], nullptr, 0, S.c, kHashMaxPb, S.dlim);
  r.post(PBNG_K_CLASSIFY);
  const Counters hc = r.readback(S.c);
  S.win_split = pick_split(r, hc.ntier[2], gr.nU);
  launch_agg<2>(r, S, hc.ntier);
  r.pre(PBNG_K_INIT);
  k_level_minlab<<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, S.part, S.cc, minlab);
  r.post(PBNG_K_INIT);
  r.pre(PBNG_K_INIT);
  k_level_label<<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, S.part, S.cc, minlab, out_comp, dn);
  r.post(PBNG_K_INIT);
  uint32_t n = 0;
  CK(cudaMemcpyAsync(&n, dn, 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  return n;
}

// Per-edge butterfly counts (Alg.1 per-edge part, kernels_edge.cuh): starts in
// U, then starts in V, each routed into three tiers; then every caller edge
// gathers accU[p] + accV[q] from its two relabeled positions.  g is oriented
// so that U is the output side.
void edge_count(const Dev& g, uint64_t* out, uint64_t* out_info, cudaStream_t s) {
  uint64_t info[4] = {0, 0, 0, 0};
  Run r(s);
  SideRank RU, RV;
  const Dev gr = relabel(r, g, RU, RV);
  uint32_t* cutU = r.alloc<uint32_t>(g.nU);
  uint32_t* cutV = r.alloc<uint32_t>(g.nV);
  uint32_t* ld = r.alloc<uint32_t>(g.nV);
  unsigned long long* cnt = r.alloc<unsigned long long>(2);  // [0] Σ d², [1] wedges
  CK(cudaMemsetAsync(cnt, 0, 16, r.st));
  r.pre(PBNG_K_EDGE);
  k_vp_cut_u<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, gr.offU, gr.adjU, RV.binoff, RV.dmax, cutU);
  r.post(PBNG_K_EDGE);
  if (g.nV) {
    r.pre(PBNG_K_EDGE);
    k_init_v<<<r.nsm * 4, 256, 0, r.st>>>(g.nV, gr.offV, ld, cnt);
    r.post(PBNG_K_EDGE);
    r.pre(PBNG_K_EDGE);
    k_vp_cut_v<<<r.nsm * 8, 256, 0, r.st>>>(g.nV, gr.offV, gr.adjV, ld, RU.binoff, RU.dmax, cutV);
    r.post(PBNG_K_EDGE);
  }
  uint64_t* accU = r.alloc<uint64_t>(g.m);
  uint64_t* accV = r.alloc<uint64_t>(g.m);
  CK(cudaMemsetAsync(accU, 0, g.m * 8, r.st));
  CK(cudaMemsetAsync(accV, 0, g.m * 8, r.st));
  const uint32_t nmax = std::max(g.nU, g.nV);
  uint2* q = r.alloc<uint2>(3ull * nmax);
  uint32_t* plen = r.alloc<uint32_t>(g.m);
  uint32_t* nq = r.alloc<uint32_t>(4);
  uint32_t* dense = nullptr;
  uint32_t ndense = 0;
  for (int side = 0; side < 2; side++) {
    EdgeArgs a;
    a.nS = side == 0 ? g.nU : g.nV;
    a.offS = side == 0 ? gr.offU : gr.offV;
    a.adjS = side == 0 ? gr.adjU : gr.adjV;
    a.offM = side == 0 ? gr.offV : gr.offU;
    a.adjM = side == 0 ? gr.adjV : gr.adjU;
    a.cutM = side == 0 ? cutV : cutU;
    a.accS = side == 0 ? accU : accV;
    a.accM = side == 0 ? accV : accU;
    a.q = q;
    a.nq = nq;
    a.wedges = cnt + 1;
    a.plen = plen;
    a.dense = nullptr;
    if (a.nS == 0) continue;
    CK(cudaMemsetAsync(nq, 0, 16, r.st));
    r.pre(PBNG_K_EDGE);
    k_edge_classify<<<r.nsm * 8, 256, 0, r.st>>>(a);
    r.post(PBNG_K_EDGE);
    uint32_t hq[4];
    CK(cudaMemcpyAsync(hq, nq, 16, cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    for (int t = 0; t < 3; t++) info[1 + t] += hq[t];
    if (hq[0]) {
      r.pre(PBNG_K_EDGE);
      k_edge_warp<<<std::min<uint32_t>(r.nsm * 5, (hq[0] + 7) / 8), kEdgeWarpThreads, edge_warp_smem(), r.st>>>(a);
      r.post(PBNG_K_EDGE);
    }
    if (hq[1]) {
      r.pre(PBNG_K_EDGE);
      k_edge_cta<<<std::min<uint32_t>(r.nsm * 2, hq[1]), kEdgeCtaThreads, edge_cta_smem(), r.st>>>(a);
      r.post(PBNG_K_EDGE);
    }
    if (hq[2]) {
      const uint32_t want = std::min<uint32_t>(r.nsm, hq[2]);
      if (a.nS > kEdgeDenseSmem && ndense < want) {  // per-CTA dense counters for start ids above the smem range
        size_t freeb = 0, totalb = 0;
        CK(cudaMemGetInfo(&freeb, &totalb));
        const uint64_t per = (uint64_t)nmax * 4;
        ndense = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, (freeb / 2) / per));
        dense = r.alloc<uint32_t>((uint64_t)ndense * nmax);
        CK(cudaMemsetAsync(dense, 0, (uint64_t)ndense * per, r.st));
      }
      a.dense = dense;
      const uint32_t grid = a.nS > kEdgeDenseSmem ? std::min(want, ndense) : want;
      r.pre(PBNG_K_EDGE);
      k_edge_dense<<<grid, kEdgeDenseThreads, edge_dense_smem(), r.st>>>(a);
      r.post(PBNG_K_EDGE);
    }
  }
  if (g.m) {
    r.pre(PBNG_K_EDGE);
    k_edge_gather<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.m, g.offU, g.adjU, RU.rank, RV.rank, gr.offU, gr.adjU,
                                                 gr.offV, gr.adjV, accU, accV, out);
    r.post(PBNG_K_EDGE);
  }
  info[0] = read_u64(r, cnt + 1);
  if (out_info) std::memcpy(out_info, info, sizeof(info));
}

// ------------------------------------------------------------ BE-Index / wing
struct BeIndex {
  uint64_t nb = 0, np = 0;
  unsigned long long* bloom_off = nullptr;
  uint32_t* bloom_k = nullptr;
  uint2* bloom_dom = nullptr;
  uint2* pair = nullptr;
  uint32_t* pair_bloom = nullptr;
};

// BE-Index of the relabeled graph gr (kernels_wing.cuh): sizes run over the
// starts of both sides, one exclusive scan over [U starts | V starts], fill run.
void be_build(Run& r, const Dev& gr, const SideRank& RU, const SideRank& RV, BeIndex& I) {
  if (gr.nU >= 0x80000000u || gr.nV >= 0x80000000u) fail(PBNG_ERR_ARG, "BE-Index needs fewer than 2^31 vertices per side");
  uint32_t* cutU = r.alloc<uint32_t>(gr.nU);
  uint32_t* cutV = r.alloc<uint32_t>(gr.nV);
  uint32_t* ld = r.alloc<uint32_t>(gr.nV);
  unsigned long long* sq = r.alloc<unsigned long long>(1);
  CK(cudaMemsetAsync(sq, 0, 8, r.st));
  r.pre(PBNG_K_EDGE);
  k_vp_cut_u<<<r.nsm * 8, 256, 0, r.st>>>(gr.nU, gr.offU, gr.adjU, RV.binoff, RV.dmax, cutU);
  r.post(PBNG_K_EDGE);
  r.pre(PBNG_K_EDGE);
  k_init_v<<<r.nsm * 4, 256, 0, r.st>>>(gr.nV, gr.offV, ld, sq);
  r.post(PBNG_K_EDGE);
  r.pre(PBNG_K_EDGE);
  k_vp_cut_v<<<r.nsm * 8, 256, 0, r.st>>>(gr.nV, gr.offV, gr.adjV, ld, RU.binoff, RU.dmax, cutV);
  r.post(PBNG_K_EDGE);
  uint32_t* mir = r.alloc<uint32_t>(gr.m);
  r.pre(PBNG_K_EDGE);
  k_be_mirror<<<r.nsm * 8, 256, 0, r.st>>>(gr.nV, gr.m, gr.offV, gr.adjV, gr.offU, gr.adjU, mir);
  r.post(PBNG_K_EDGE);
  const uint32_t nmax = std::max(gr.nU, gr.nV);
  size_t freeb = 0, totalb = 0;
  CK(cudaMemGetInfo(&freeb, &totalb));
  const uint32_t ctas = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>({(uint64_t)r.nsm * 4, (uint64_t)nmax, (freeb / 4) / (12ull * nmax)}));
  uint32_t* cnt = r.alloc<uint32_t>((uint64_t)ctas * nmax);
  uint32_t* bidx = r.alloc<uint32_t>((uint64_t)ctas * nmax);
  uint32_t* pbase = r.alloc<uint32_t>((uint64_t)ctas * nmax);
  CK(cudaMemsetAsync(cnt, 0, (uint64_t)ctas * nmax * 4, r.st));
  CK(cudaMemsetAsync(bidx, 0xFF, (uint64_t)ctas * nmax * 4, r.st));
  const uint64_t nsz = (uint64_t)gr.nU + 1 + gr.nV + 1;
  unsigned long long* nbs = r.alloc<unsigned long long>(nsz);
  unsigned long long* nps = r.alloc<unsigned long long>(nsz);
  CK(cudaMemsetAsync(nbs, 0, nsz * 8, r.st));
  CK(cudaMemsetAsync(nps, 0, nsz * 8, r.st));
  uint32_t* ticket = r.alloc<uint32_t>(1);
  auto args = [&](int side) {
    BeArgs b;
    std::memset(&b, 0, sizeof(b));
    EdgeArgs& a = b.a;
    a.nS = side == 0 ? gr.nU : gr.nV;
    a.offS = side == 0 ? gr.offU : gr.offV;
    a.adjS = side == 0 ? gr.adjU : gr.adjV;
    a.offM = side == 0 ? gr.offV : gr.offU;
    a.adjM = side == 0 ? gr.adjV : gr.adjU;
    a.cutM = side == 0 ? cutV : cutU;
    b.mirM2U = mir;
    b.mirS2U = mir;
    b.side = (uint32_t)side;
    b.cnt = cnt;
    b.bidx = bidx;
    b.pbase = pbase;
    const uint64_t o = side == 0 ? 0 : (uint64_t)gr.nU + 1;
    b.nb_s = nbs + o;
    b.np_s = nps + o;
    b.bS = nbs + o;
    b.pS = nps + o;
    b.ticket = ticket;
    return b;
  };
  for (int side = 0; side < 2; side++) {
    BeArgs b = args(side);
    if (!b.a.nS) continue;
    CK(cudaMemsetAsync(ticket, 0, 4, r.st));
    r.pre(PBNG_K_EDGE);
    k_be_build<false><<<std::min<uint32_t>(ctas, b.a.nS), kBeThreads, 0, r.st>>>(b);
    r.post(PBNG_K_EDGE);
  }
  scan_u64(r, nbs, nsz);
  scan_u64(r, nps, nsz);
  // totals: the scan's last entry is the sum of everything before it (its own input is 0)
  I.nb = read_u64(r, nbs + nsz - 1);
  I.np = read_u64(r, nps + nsz - 1);
  if (I.np >= 0xFFFFFFFFull) fail(PBNG_ERR_OOM, "BE-Index has 2^32 or more twin pairs");
  I.bloom_off = r.alloc<unsigned long long>(I.nb + 1);
  I.bloom_k = r.alloc<uint32_t>(I.nb);
  I.bloom_dom = r.alloc<uint2>(I.nb);
  I.pair = r.alloc<uint2>(I.np);
  I.pair_bloom = r.alloc<uint32_t>(I.np);
  CK(cudaMemcpyAsync(I.bloom_off + I.nb, &I.np, 8, cudaMemcpyHostToDevice, r.st));
  for (int side = 0; side < 2; side++) {
    BeArgs b = args(side);
    if (!b.a.nS) continue;
    b.bloom_off = I.bloom_off;
    b.bloom_k = I.bloom_k;
    b.bloom_dom = I.bloom_dom;
    b.pair = I.pair;
    b.pair_bloom = I.pair_bloom;
    CK(cudaMemsetAsync(ticket, 0, 4, r.st));
    r.pre(PBNG_K_EDGE);
    k_be_build<true><<<std::min<uint32_t>(ctas, b.a.nS), kBeThreads, 0, r.st>>>(b);
    r.post(PBNG_K_EDGE);
  }
  CK(cudaStreamSynchronize(r.st));  // &I.np must outlive its copy
}

// Wing decomposition of gr on its BE-Index (kernels_wing.cuh): θ per canonical edge id.
void wing_peel(Run& r, const Dev& gr, const BeIndex& I, uint64_t* theta, uint64_t* info) {
  const uint64_t m = gr.m;
  WingArgs w;
  std::memset(&w, 0, sizeof(w));
  w.m = m;
  w.nb = I.nb;
  w.bloom_off = I.bloom_off;
  w.bloom_k = I.bloom_k;
  w.pair = I.pair;
  w.pair_bloom = I.pair_bloom;
  w.theta = theta;
  w.bloom_d = r.alloc<uint32_t>(I.nb);
  CK(cudaMemsetAsync(w.bloom_d, 0, I.nb * 4, r.st));
  w.pstate = r.alloc<uint32_t>(I.np);
  CK(cudaMemsetAsync(w.pstate, 0, I.np * 4, r.st));
  w.sup = r.alloc<unsigned long long>(m);
  CK(cudaMemsetAsync(w.sup, 0, m * 8, r.st));
  unsigned long long* ioff = r.alloc<unsigned long long>(m + 1);
  unsigned long long* cur = r.alloc<unsigned long long>(m + 1);
  CK(cudaMemsetAsync(ioff, 0, (m + 1) * 8, r.st));
  uint32_t* inc = r.alloc<uint32_t>(2 * I.np);
  if (I.np) {
    r.pre(PBNG_K_FD);
    k_wing_init<<<r.nsm * 8, 256, 0, r.st>>>(w);
    r.post(PBNG_K_FD);
    r.pre(PBNG_K_FD);
    k_wing_inc_count<<<r.nsm * 8, 256, 0, r.st>>>(w, ioff);
    r.post(PBNG_K_FD);
  }
  scan_u64(r, ioff, m + 1);
  CK(cudaMemcpyAsync(cur, ioff, (m + 1) * 8, cudaMemcpyDeviceToDevice, r.st));
  if (I.np) {
    r.pre(PBNG_K_FD);
    k_wing_inc_fill<<<r.nsm * 8, 256, 0, r.st>>>(w, cur, inc);
    r.post(PBNG_K_FD);
  }
  w.inc_off = ioff;
  w.inc = inc;
  w.alive = r.alloc<uint8_t>(m);
  CK(cudaMemsetAsync(w.alive, 1, m, r.st));
  uint32_t* live[2] = {r.alloc<uint32_t>(m), r.alloc<uint32_t>(m)};
  r.pre(PBNG_K_FD);
  k_iota<<<r.nsm * 8, 256, 0, r.st>>>(m, live[0]);
  r.post(PBNG_K_FD);
  uint32_t* SX[2] = {r.alloc<uint32_t>(m), r.alloc<uint32_t>(m)};
  w.T = r.alloc<uint32_t>(std::max<uint64_t>(I.nb, 1));
  if (!std::getenv("PBNG_WING_HOST")) {
    // device-driven peel: one persistent cooperative launch (k_wing_peel);
    // PBNG_WING_HOST=1 keeps the host-driven rounds below (same phases, for A/B runs)
    WingDev* dc = r.alloc<WingDev>(1);
    WingDev init;
    std::memset(&init, 0, sizeof(init));
    init.minsup = ~0ull;
    init.minC = ~0ull;
    CK(cudaMemcpyAsync(dc, &init, sizeof(init), cudaMemcpyHostToDevice, r.st));
    uint32_t* cand[2] = {r.alloc<uint32_t>(m), r.alloc<uint32_t>(m)};  // candidate band lists
    void* args[] = {&w, &live[0], &live[1], &SX[0], &SX[1], &cand[0], &cand[1], &dc};
    r.pre(PBNG_K_FD);
    CK(cudaLaunchCooperativeKernel((const void*)k_wing_peel, dim3(r.nsm), dim3(kWingThreads), args, 0, r.st));
    r.post(PBNG_K_FD);
    WingDev out;
    CK(cudaMemcpyAsync(&out, dc, sizeof(out), cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    if (info) {
      info[0] = I.nb;
      info[1] = I.np;
      info[2] = out.levels;
      info[3] = out.rounds;
    }
    if (std::getenv("PBNG_TRACE"))
      std::fprintf(stderr, "wing peel cycles (CTA 0): scan=%llu select=%llu claim=%llu update=%llu\n", out.clk[0],
                   out.clk[1], out.clk[2], out.clk[3]);
    return;
  }
  w.ctl = r.alloc<WingCtl>(1);
  WingCtl* hctl = nullptr;
  CK(cudaMallocHost(&hctl, sizeof(WingCtl)));
  struct HostFree {
    WingCtl* p;
    ~HostFree() { cudaFreeHost(p); }
  } hf{hctl};
  uint64_t k = 0, levels = 0, rounds = 0;
  uint32_t nlive = (uint32_t)m, cur_live = 0;
  const WingCtl zero{0, 0, 0, 0, ~0ull};
  for (;;) {
    // level scan: compact the live list, minimum live support
    CK(cudaMemcpyAsync(w.ctl, &zero, sizeof(WingCtl), cudaMemcpyHostToDevice, r.st));
    w.live = live[cur_live];
    r.pre(PBNG_K_FD);
    k_wing_scan<<<std::max<uint32_t>(1, std::min<uint32_t>(r.nsm * 8, (nlive + 255) / 256)), 256, 0, r.st>>>(
        w, nlive, live[cur_live], live[cur_live ^ 1]);
    r.post(PBNG_K_FD);
    CK(cudaMemcpyAsync(hctl, w.ctl, sizeof(WingCtl), cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    cur_live ^= 1;
    nlive = hctl->nlive;
    if (nlive == 0) break;
    k = std::max<uint64_t>(k, hctl->minsup);
    levels++;
    w.live = live[cur_live];
    w.S = SX[0];
    CK(cudaMemsetAsync(&w.ctl->nS, 0, 4, r.st));
    r.pre(PBNG_K_FD);
    k_wing_select<<<std::min<uint32_t>(r.nsm * 8, (nlive + 255) / 256), 256, 0, r.st>>>(w, nlive, k);
    r.post(PBNG_K_FD);
    CK(cudaMemcpyAsync(hctl, w.ctl, sizeof(WingCtl), cudaMemcpyDeviceToHost, r.st));
    CK(cudaStreamSynchronize(r.st));
    uint32_t nS = hctl->nS;
    int cs = 0;
    while (nS) {
      rounds++;
      w.S = SX[cs];
      w.X = SX[cs ^ 1];
      CK(cudaMemsetAsync(&w.ctl->nX, 0, 8, r.st));  // nX, nT
      r.pre(PBNG_K_FD);
      k_wing_claim<<<std::min<uint32_t>(r.nsm * 8, (nS + 7) / 8), 256, 0, r.st>>>(w, nS, k);
      r.post(PBNG_K_FD);
      r.pre(PBNG_K_FD);
      k_wing_kill<<<std::min<uint32_t>(r.nsm * 8, (nS + 255) / 256), 256, 0, r.st>>>(w, nS);
      r.post(PBNG_K_FD);
      CK(cudaMemcpyAsync(hctl, w.ctl, sizeof(WingCtl), cudaMemcpyDeviceToHost, r.st));
      CK(cudaStreamSynchronize(r.st));
      const uint32_t nT = hctl->nT;
      if (nT) {
        r.pre(PBNG_K_FD);
        k_wing_update<<<std::min<uint32_t>(r.nsm * 8, (nT + 7) / 8), 256, 0, r.st>>>(w, nT, k);
        r.post(PBNG_K_FD);
      }
      CK(cudaMemcpyAsync(hctl, w.ctl, sizeof(WingCtl), cudaMemcpyDeviceToHost, r.st));
      CK(cudaStreamSynchronize(r.st));
      nS = hctl->nX;
      cs ^= 1;
    }
  }
  if (info) {
    info[0] = I.nb;
    info[1] = I.np;
    info[2] = levels;
    info[3] = rounds;
  }
}

void wing_decompose(const Dev& g, uint64_t* out, uint64_t* info, cudaStream_t s) {
  Run r(s);
  SideRank RU, RV;
  const Dev gr = relabel(r, g, RU, RV);
  const bool trace = std::getenv("PBNG_TRACE") != nullptr;  // phase times on stderr (development aid)
  cudaEvent_t t0 = trace ? r.event() : nullptr;
  BeIndex I;
  be_build(r, gr, RU, RV, I);
  cudaEvent_t t1 = trace ? r.event() : nullptr;
  uint64_t* theta = r.alloc<uint64_t>(g.m);
  wing_peel(r, gr, I, theta, info);
  if (trace) {
    cudaEvent_t t2 = r.event();
    CK(cudaStreamSynchronize(r.st));
    std::fprintf(stderr, "wing: be_index_ms=%.3f peel_ms=%.3f blooms=%llu pairs=%llu\n", elapsed(t0, t1), elapsed(t1, t2),
                 (unsigned long long)I.nb, (unsigned long long)I.np);
  }
  r.pre(PBNG_K_INIT);
  k_wing_gather<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.m, g.offU, g.adjU, RU.rank, RV.rank, gr.offU, gr.adjU, theta,
                                              out);
  r.post(PBNG_K_INIT);
  CK(cudaStreamSynchronize(r.st));
}

void be_index_export(const Dev& g, uint64_t* sizes, unsigned long long* bloom_off, uint32_t* bloom_k,
                     uint32_t* dom, uint32_t* pairs, cudaStream_t s) {
  Run r(s);
  SideRank RU, RV;
  const Dev gr = relabel(r, g, RU, RV);
  BeIndex I;
  be_build(r, gr, RU, RV, I);
  sizes[0] = I.nb;
  sizes[1] = I.np;
  if (!bloom_off) return;  // size query
  uint32_t* r2c = r.alloc<uint32_t>(g.m);
  r.pre(PBNG_K_INIT);
  k_edge_r2c<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.m, g.offU, g.adjU, RU.rank, RV.rank, gr.offU, gr.adjU, r2c);
  r.post(PBNG_K_INIT);
  CK(cudaMemcpyAsync(bloom_off, I.bloom_off, (I.nb + 1) * 8, cudaMemcpyDeviceToDevice, r.st));
  if (I.nb) CK(cudaMemcpyAsync(bloom_k, I.bloom_k, I.nb * 4, cudaMemcpyDeviceToDevice, r.st));
  if (I.nb || I.np) {
    r.pre(PBNG_K_INIT);
    k_be_export<<<r.nsm * 8, 256, 0, r.st>>>(I.nb, I.np, I.pair, r2c, I.bloom_dom, RU.inv, RV.inv, pairs, dom);
    r.post(PBNG_K_INIT);
  }
  CK(cudaStreamSynchronize(r.st));
}

template <class Fn>
int guarded(Fn&& fn) {
  g_err.clear();
  try {
    fn();
    if (PBNG_CHECK) {
      unsigned int line = 0;
      CK(cudaMemcpyFromSymbol(&line, g_check_line, sizeof(line)));
      if (line) {
        const unsigned int zero = 0;
        CK(cudaMemcpyToSymbol(g_check_line, &zero, sizeof(zero)));
        fail(PBNG_ERR_CUDA, "device check failed (PBNG_DCHECK) at kernel source line " + std::to_string(line));
      }
    }
    return PBNG_OK;
  } catch (const Fail& f) {
    return f.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return PBNG_ERR_OOM;
  } catch (...) {
    g_err = "unexpected exception";
    return PBNG_ERR_CUDA;
  }
}

}  // namespace

extern "C" {

int pbng_count_butterflies(pbng_csr U, pbng_csr V, int side, uint64_t* out_support, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, side, g);
    if (!out_support && g.nU) fail(PBNG_ERR_ARG, "out_support is null");
    if (g.nU == 0) return;
    Run r((cudaStream_t)stream);
    State S;
    SideRank RU, RV;
    const Dev gr = relabel(r, g, RU, RV);
    alloc_state(r, S, gr, false, RU, RV, true);
    count_live(r, S);
    r.pre(PBNG_K_INIT);
    k_gather<uint64_t><<<r.nsm * 4, 256, 0, r.st>>>(g.nU, RU.rank, S.support, out_support);
    r.post(PBNG_K_INIT);
    CK(cudaStreamSynchronize(r.st));
  });
}

int pbng_count_edge_butterflies(pbng_csr U, pbng_csr V, int side, uint64_t* out_edge_support,
                                uint64_t* out_info, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, side, g);
    if (out_info) std::memset(out_info, 0, 4 * sizeof(uint64_t));
    if (!out_edge_support && g.m) fail(PBNG_ERR_ARG, "out_edge_support is null");
    if (g.m == 0) return;
    edge_count(g, out_edge_support, out_info, (cudaStream_t)stream);
  });
}

int pbng_be_index(pbng_csr U, pbng_csr V, uint64_t* out_sizes, uint64_t* bloom_off, uint32_t* bloom_k,
                  uint32_t* bloom_dom, uint32_t* pairs, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, 0, g);
    if (!out_sizes) fail(PBNG_ERR_ARG, "out_sizes is null");
    out_sizes[0] = out_sizes[1] = 0;
    if (bloom_off && !(bloom_k && bloom_dom && pairs)) fail(PBNG_ERR_ARG, "null BE-Index output");
    if (g.m == 0) {
      if (bloom_off) CK(cudaMemsetAsync(bloom_off, 0, 8, (cudaStream_t)stream));
      CK(cudaStreamSynchronize((cudaStream_t)stream));
      return;
    }
    be_index_export(g, out_sizes, (unsigned long long*)bloom_off, bloom_k, bloom_dom, pairs, (cudaStream_t)stream);
  });
}

int pbng_wing_decompose(pbng_csr U, pbng_csr V, int side, uint64_t* out_theta, uint64_t* out_info, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, side, g);
    if (out_info) std::memset(out_info, 0, 4 * sizeof(uint64_t));
    if (!out_theta && g.m) fail(PBNG_ERR_ARG, "out_theta is null");
    if (g.m == 0) return;
    wing_decompose(g, out_theta, out_info, (cudaStream_t)stream);
  });
}

int pbng_tip_decompose(pbng_csr U, pbng_csr V, int side, uint32_t P, uint64_t* out_tip, uint32_t opts,
                       pbng_stats* stats, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, side, g);
    if (!out_tip && g.nU) fail(PBNG_ERR_ARG, "out_tip is null");
    Out o;
    o.tip = out_tip;
    decompose(g, P, opts, o, stats, (cudaStream_t)stream);
  });
}

int pbng_tip_plan(pbng_csr U, pbng_csr V, int side, uint32_t P, uint32_t opts, uint32_t* out_part,
                  uint64_t* out_init, uint64_t* out_bounds, uint32_t* out_nparts, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, side, g);
    if (!out_bounds || !out_nparts || (g.nU && (!out_part || !out_init))) fail(PBNG_ERR_ARG, "null output");
    Out o;
    o.part = out_part;
    o.init = out_init;
    o.bounds = out_bounds;
    o.nparts = out_nparts;
    decompose(g, P, opts, o, nullptr, (cudaStream_t)stream);
  });
}

int pbng_tip_decompose_host(pbng_csr U, pbng_csr V, int side, uint32_t P, uint64_t* out_tip, uint32_t opts,
                            pbng_stats* stats, void* stream) {
  return guarded([&] {
    if (U.m != V.m) fail(PBNG_ERR_ARG, "U.m != V.m");
    if (!U.offsets || !V.offsets || (U.m && (!U.indices || !V.indices))) fail(PBNG_ERR_ARG, "null CSR pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t nOut = side == 1 ? V.n : U.n;
    if (!out_tip && nOut) fail(PBNG_ERR_ARG, "out_tip is null");
    // device copies (freed by the Run destructor)
    Run r(s);
    uint64_t* dou = r.alloc<uint64_t>((size_t)U.n + 1);
    uint64_t* dov = r.alloc<uint64_t>((size_t)V.n + 1);
    uint32_t* dau = r.alloc<uint32_t>(U.m);
    uint32_t* dav = r.alloc<uint32_t>(V.m);
    uint64_t* dtip = r.alloc<uint64_t>(nOut);
    CK(cudaMemcpyAsync(dou, U.offsets, ((size_t)U.n + 1) * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dov, V.offsets, ((size_t)V.n + 1) * 8, cudaMemcpyHostToDevice, s));
    if (U.m) {
      CK(cudaMemcpyAsync(dau, U.indices, U.m * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dav, V.indices, V.m * 4, cudaMemcpyHostToDevice, s));
    }
    pbng_csr du{dou, dau, U.n, U.m}, dv{dov, dav, V.n, V.m};
    Dev g;
    orient(du, dv, side, g);
    Out o;
    o.tip = dtip;
    decompose(g, P, opts, o, stats, s);
    if (nOut) CK(cudaMemcpyAsync(out_tip, dtip, (size_t)nOut * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int pbng_tip_components(pbng_csr U, pbng_csr V, int side, const uint64_t* tip, uint64_t k, uint32_t* out_comp,
                        uint32_t* out_ncomp, void* stream) {
  return guarded([&] {
    Dev g;
    orient(U, V, side, g);
    if (!out_ncomp || (g.nU && (!tip || !out_comp))) fail(PBNG_ERR_ARG, "null pointer");
    *out_ncomp = 0;
    if (g.nU == 0) return;
    *out_ncomp = tip_level(g, tip, k, out_comp, (cudaStream_t)stream);
  });
}

int pbng_kernel_times(float* out_ms) {
  return guarded([&] {
    if (!out_ms) fail(PBNG_ERR_ARG, "out_ms is null");
    for (int i = 0; i < PBNG_K_NUM; i++) out_ms[i] = 0.0f;
    for (const DeferredSpan& sp : deferred_spans()) {
      float ms = 0;
      CK(cudaEventSynchronize(sp.b));
      CK(cudaEventElapsedTime(&ms, sp.a, sp.b));
      out_ms[sp.kind] += ms;
      event_pool().push_back(sp.a);
      event_pool().push_back(sp.b);
    }
    deferred_spans().clear();
  });
}

int pbng_release_memory(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(g_dev_mu);
    for (int d = 0; d < kMaxDevices; d++)
      if (g_dev_ready[d]) CK(cudaMemPoolTrimTo(g_dev_pool[d], 0));
  });
}

const char* pbng_last_error(void) { return g_err.c_str(); }

const char* pbng_version(void) { return "pbng-b200 0.1 sm_100a"; }

}  // extern "C"
