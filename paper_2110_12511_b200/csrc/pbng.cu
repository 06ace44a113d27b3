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
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pbng.h"
#include "kernels_fd.cuh"

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
size_t range_smem() { return sizeof(RangeSmem); }
size_t hist_smem() { return (size_t)kBins * 12; }
size_t fd_smem() { return ((size_t)(kFdThreads / 32) * 2 * kFdWarpSlots + 2 * kCtaSlots + kFdThreads) * 4; }

void set_attrs_once() {
  static std::once_flag once;
  std::call_once(once, [] {
    // keep stream-ordered scratch cached between calls (no re-mapping per decomposition)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaFuncSetAttribute(k_agg_warp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_range<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)range_smem());
    cudaFuncSetAttribute(k_agg_range<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)range_smem());
    cudaFuncSetAttribute(k_range_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist_smem());
    cudaFuncSetAttribute(k_fd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fd_smem());
    cudaGetLastError();
  });
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

class Run {
 public:
  explicit Run(cudaStream_t s) : st(s) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    set_attrs_once();
    CK(cudaMallocHost(&hc, sizeof(Counters)));
  }
  ~Run() {
    for (void* p : allocs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (hc) cudaFreeHost(hc);
    cudaGetLastError();
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st);
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
    CK(cudaEventCreate(&e));
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
      CK(cudaEventCreate(&pending));
      CK(cudaEventRecord(pending, st));
    }
  }
  void post(int kind) {
    check(cudaGetLastError(), "kernel launch", kind);
    launches++;
    if (timing) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      CK(cudaEventRecord(e, st));
      spans.push_back({kind, pending, e});
      events.push_back(pending);
      events.push_back(e);
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
  int nsm = 148;
  Counters* hc = nullptr;
  bool timing = false;
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
  uint2* tier[3];
  uint32_t* vflag;
  uint32_t* touched;
  Counters* c;
  unsigned long long* hist_w;
  uint32_t* hist_n;
  unsigned long long* sum_d2;
  uint32_t nslots;
  uint32_t *slot_cnt, *slot_touch, *slot_dup;  // FD heavy path: dense counters per CTA
  uint64_t piece_cap;                          // tier-1 cursor scratch per CTA
  uint64_t *piece_pos, *piece_end, *piece_save;
  uint32_t* piece_head;
  uint32_t* piece_srange;
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

void alloc_state(Run& r, State& S, const Dev& g, bool need_live) {
  S.g = g;
  S.ld = r.alloc<uint32_t>(g.nV);
  S.adjL = need_live ? r.alloc<uint32_t>(g.m) : const_cast<uint32_t*>(g.adjV);
  S.tmp = need_live ? r.alloc<uint32_t>(g.m) : nullptr;
  S.wc = r.alloc<uint64_t>(g.nU);
  S.support = r.alloc<uint64_t>(g.nU);
  S.init = need_live ? r.alloc<uint64_t>(g.nU) : nullptr;
  S.part = r.alloc<uint32_t>(g.nU);
  S.F = r.alloc<uint32_t>(g.nU);
  for (int t = 0; t < 3; t++) S.tier[t] = r.alloc<uint2>(g.nU);
  S.vflag = r.alloc<uint32_t>(g.nV);
  S.touched = r.alloc<uint32_t>(g.nV);
  S.c = r.alloc<Counters>(1);
  S.hist_w = r.alloc<unsigned long long>(kBins);
  S.hist_n = r.alloc<uint32_t>(kBins);
  S.sum_d2 = r.alloc<unsigned long long>(1);
  CK(cudaMemsetAsync(S.vflag, 0, (size_t)std::max<uint32_t>(g.nV, 1) * 4, r.st));
  CK(cudaMemsetAsync(S.c, 0, sizeof(Counters), r.st));
  CK(cudaMemsetAsync(S.sum_d2, 0, 8, r.st));
  if (need_live && g.m) CK(cudaMemcpyAsync(S.adjL, g.adjV, g.m * 4, cudaMemcpyDeviceToDevice, r.st));
  r.pre(PBNG_K_INIT);
  k_init_v<<<r.nsm * 4, 256, 0, r.st>>>(g.nV, g.offV, S.ld, S.sum_d2);
  r.post(PBNG_K_INIT);
  unsigned long long* dmax = r.alloc<unsigned long long>(1);
  CK(cudaMemsetAsync(dmax, 0, 8, r.st));
  r.pre(PBNG_K_INIT);
  k_init_u<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.offU, g.adjU, g.offV, S.wc, S.part, dmax);
  r.post(PBNG_K_INIT);
  unsigned long long hmax = 0;
  CK(cudaMemcpyAsync(&hmax, dmax, 8, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  S.piece_cap = std::max<unsigned long long>(hmax, 1);
  const size_t np = (size_t)r.nsm * kRangeCtas * S.piece_cap;
  S.piece_pos = r.alloc<uint64_t>(np);
  S.piece_end = r.alloc<uint64_t>(np);
  S.piece_save = r.alloc<uint64_t>(np);
  S.piece_head = r.alloc<uint32_t>(np);
  S.piece_srange = r.alloc<uint32_t>(np);
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
  a.piece_pos = S.piece_pos;
  a.piece_end = S.piece_end;
  a.piece_save = S.piece_save;
  a.piece_head = S.piece_head;
  a.piece_srange = S.piece_srange;
  a.piece_cap = S.piece_cap;
  a.c = S.c;
  return a;
}

template <int MODE>
void launch_agg(Run& r, const State& S) {
  r.pre(PBNG_K_AGG_WARP);
  k_agg_warp<MODE><<<r.nsm * 3, kWarpTierThreads, warp_tier_smem(), r.st>>>(agg_args(S, 0));
  r.post(PBNG_K_AGG_WARP);
  r.pre(PBNG_K_AGG_CTA);
  k_agg_range<MODE><<<r.nsm * kRangeCtas, kRangeThreads, range_smem(), r.st>>>(agg_args(S, 1));
  r.post(PBNG_K_AGG_CTA);
}

void reset_tiers(Run& r, State& S) {
  CK(cudaMemsetAsync(&S.c->ntier[0], 0, 7 * sizeof(uint32_t), r.st));  // ntier[3] + ticket[4]
}

// Butterfly count of every unassigned u (initial count, and §5.1 re-count).
void count_live(Run& r, State& S) {
  reset_tiers(r, S);
  r.pre(PBNG_K_CLASSIFY);
  k_classify<0><<<r.nsm * 8, 256, 0, r.st>>>(S.g.nU, nullptr, nullptr, S.g.offU, S.g.adjU, S.ld, S.part,
                                               S.support, S.tier[0], S.tier[1], S.tier[2], nullptr, 0, S.c);
  r.post(PBNG_K_CLASSIFY);
  launch_agg<0>(r, S);
}

void compact(Run& r, State& S, uint32_t epoch) {
  const uint32_t big = 4096;
  CK(cudaMemsetAsync(&S.c->ntouched, 0, 4, r.st));
  r.pre(PBNG_K_COMPACT);
  k_collect_touched<<<r.nsm * 8, 256, 0, r.st>>>(S.g.nV, S.vflag, epoch, S.touched, S.c);
  r.post(PBNG_K_COMPACT);
  r.pre(PBNG_K_COMPACT);
  k_compact<<<r.nsm * 8, 256, 0, r.st>>>(S.touched, &S.c->ntouched, S.g.offV, S.adjL, S.tmp, S.ld, S.part, big,
                                         S.c);
  r.post(PBNG_K_COMPACT);
  r.pre(PBNG_K_COMPACT);
  k_compact_big<<<r.nsm, 512, 0, r.st>>>(S.touched, &S.c->ntouched, S.g.offV, S.adjL, S.tmp, S.ld, S.part, big,
                                         S.c);
  r.post(PBNG_K_COMPACT);
}

struct Plan {
  std::vector<uint64_t> bounds;  // bounds[0] = 0 ... bounds[nparts] = inf
  uint32_t nparts = 0;
};

// Coarse-grained decomposition (Alg.4 structure P:799-816, tip P:982-991).
void run_cd(Run& r, State& S, uint32_t P, uint32_t opts, Plan& plan, pbng_stats& st) {
  const bool del = !(opts & PBNG_OPT_NO_DELETE);
  const uint32_t nU = S.g.nU;
  std::vector<unsigned long long> hw(kBins);
  std::vector<uint32_t> hn(kBins);
  unsigned long long sum_d2 = 0;
  CK(cudaMemcpyAsync(&sum_d2, S.sum_d2, 8, cudaMemcpyDeviceToHost, r.st));
  plan.bounds.assign(1, 0);
  double scale = 1.0;  // two-way adaptive target, second adaptation
  uint32_t epoch = 0;
  for (uint32_t pid = 0; pid < P; pid++) {
    // --- partition start: ⋈^init snapshot + weighted support histogram
    CK(cudaMemsetAsync(S.hist_w, 0, kBins * 8, r.st));
    CK(cudaMemsetAsync(S.hist_n, 0, kBins * 4, r.st));
    CK(cudaMemsetAsync(&S.c->live_wc, 0, 16, r.st));
    r.pre(PBNG_K_RANGE);
    k_range_hist<<<r.nsm, 1024, hist_smem(), r.st>>>(nU, S.part, S.support, S.wc, S.init, S.hist_w, S.hist_n,
                                                     S.c);
    r.post(PBNG_K_RANGE);
    CK(cudaMemcpyAsync(hw.data(), S.hist_w, kBins * 8, cudaMemcpyDeviceToHost, r.st));
    CK(cudaMemcpyAsync(hn.data(), S.hist_n, kBins * 4, cudaMemcpyDeviceToHost, r.st));
    const Counters hc0 = r.readback(S.c);
    if (hc0.live_n == 0) break;
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
                                                   S.tier[0], S.tier[1], S.tier[2], S.vflag, epoch, S.c);
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
      const unsigned long long recount_cost = sum_d2 - hc.ld2_drop;  // one-sided re-count cost (g10)
      const bool recount = !(opts & PBNG_OPT_NO_RECOUNT) &&
                           ((opts & PBNG_OPT_FORCE_RECOUNT) || hc.wedges > recount_cost);
      if (recount) {
        // §5.1: re-compute supports of all remaining vertices
        if (del) compact(r, S, epoch);
        count_live(r, S);
        st.recounts++;
      } else {
        launch_agg<1>(r, S);
        if (del) compact(r, S, epoch);
      }
    }
    if (!del) compact(r, S, epoch);
    scale = part_wc ? (double)first_wc / (double)part_wc : 1.0;
  }
  plan.nparts = (uint32_t)plan.bounds.size() - 1;
  if (plan.nparts) plan.bounds.back() = kInf;
}

// Fine-grained decomposition -> theta.
void run_fd(Run& r, State& S, const Plan& plan, uint64_t* theta, pbng_stats& st, float& ms_build) {
  const uint32_t np = plan.nparts, nU = S.g.nU;
  cudaEvent_t e0 = r.event();
  uint32_t* pcount = r.alloc<uint32_t>(np);
  uint32_t* poff = r.alloc<uint32_t>(np + 1);
  uint32_t* pcur = r.alloc<uint32_t>(np);
  unsigned long long* work = r.alloc<unsigned long long>(np);
  uint32_t* order = r.alloc<uint32_t>(np);
  uint32_t* members = r.alloc<uint32_t>(nU);
  uint32_t* sel = r.alloc<uint32_t>(nU);
  uint32_t* selpb = r.alloc<uint32_t>(nU);
  uint32_t* fstate = r.alloc<uint32_t>(nU);
  uint32_t* cand = r.alloc<uint32_t>(nU);
  uint32_t* bigl = r.alloc<uint32_t>(nU);
  uint64_t* seg = r.alloc<uint64_t>(S.g.m);
  unsigned long long* fdc = r.alloc<unsigned long long>(3);  // wedges, updates, steps
  uint32_t* misc = r.alloc<uint32_t>(3);                     // ticket, rounds_max, heavy count
  CK(cudaMemsetAsync(pcount, 0, (size_t)np * 4, r.st));
  CK(cudaMemsetAsync(pcur, 0, (size_t)np * 4, r.st));
  CK(cudaMemsetAsync(work, 0, (size_t)np * 8, r.st));
  CK(cudaMemsetAsync(fstate, 0, (size_t)nU * 4, r.st));
  CK(cudaMemsetAsync(fdc, 0, 24, r.st));
  CK(cudaMemsetAsync(misc, 0, 12, r.st));
  r.pre(PBNG_K_FD_BUILD);
  k_part_count<<<r.nsm * 4, 256, np * 4, r.st>>>(nU, S.part, np, pcount);
  r.post(PBNG_K_FD_BUILD);
  std::vector<uint32_t> hcount(np), hoff(np + 1);
  CK(cudaMemcpyAsync(hcount.data(), pcount, (size_t)np * 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  hoff[0] = 0;
  for (uint32_t i = 0; i < np; i++) hoff[i + 1] = hoff[i] + hcount[i];
  CK(cudaMemcpyAsync(poff, hoff.data(), (size_t)(np + 1) * 4, cudaMemcpyHostToDevice, r.st));
  r.pre(PBNG_K_FD_BUILD);
  k_part_scatter<<<r.nsm * 8, 256, 0, r.st>>>(nU, S.part, poff, pcur, members);
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
  std::vector<uint32_t> ord(np);
  for (uint32_t i = 0; i < np; i++) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return hwork[a] > hwork[b]; });
  CK(cudaMemcpyAsync(order, ord.data(), (size_t)np * 4, cudaMemcpyHostToDevice, r.st));
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
  a.order = order;
  a.nparts = np;
  a.ticket = misc;
  a.members = members;
  a.sel = sel;
  a.selpb = selpb;
  a.s = S.support;
  a.state = fstate;
  a.cand = cand;
  a.bigl = bigl;
  a.theta = theta;
  a.slot_cnt = S.slot_cnt;
  a.slot_touch = S.slot_touch;
  a.slot_dup = S.slot_dup;
  a.wedges = fdc;
  a.updates = fdc + 1;
  a.rounds_max = misc + 1;
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>({np, (uint32_t)r.nsm, S.nslots}));
  r.pre(PBNG_K_FD);
  k_fd<<<grid, kFdThreads, fd_smem(), r.st>>>(a);
  r.post(PBNG_K_FD);
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
  r.timing = (opts & PBNG_OPT_STATS) != 0;
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
  cudaEvent_t t0 = r.event();
  alloc_state(r, S, g, true);
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
  st.wedges_cd = c1.cum_wedges - c0.cum_wedges;
  for (int i = 0; i < 4; i++) st.impl[i] = c1.dbg[i];
  st.uv_steps += c1.cum_steps;
  st.ms_count = elapsed(t0, t1);
  st.ms_cd = elapsed(t1, t2);
  if (out.part) {
    CK(cudaMemcpyAsync(out.part, S.part, (size_t)g.nU * 4, cudaMemcpyDeviceToDevice, r.st));
    CK(cudaMemcpyAsync(out.init, S.init, (size_t)g.nU * 8, cudaMemcpyDeviceToDevice, r.st));
    for (uint32_t i = 0; i <= P; i++) out.bounds[i] = i < plan.bounds.size() ? plan.bounds[i] : kInf;
    *out.nparts = plan.nparts;
    CK(cudaStreamSynchronize(r.st));
  }
  if (out.tip) {
    float ms_build = 0;
    run_fd(r, S, plan, out.tip, st, ms_build);
    st.ms_fd_build = ms_build;
  }
  CK(cudaStreamSynchronize(r.st));
  st.launches = r.launches;
  if (r.timing) r.kernel_ms(st.ms_kernel);
  if (stats) *stats = st;
}

template <class Fn>
int guarded(Fn&& fn) {
  g_err.clear();
  try {
    fn();
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
    alloc_state(r, S, g, false);
    count_live(r, S);
    CK(cudaMemcpyAsync(out_support, S.support, (size_t)g.nU * 8, cudaMemcpyDeviceToDevice, r.st));
    CK(cudaStreamSynchronize(r.st));
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

const char* pbng_last_error(void) { return g_err.c_str(); }

const char* pbng_version(void) { return "pbng-b200 0.1 sm_100a"; }

}  // extern "C"
