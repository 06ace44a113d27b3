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
#define LAUNCHED(name) check(cudaGetLastError(), "launch " name, __LINE__)

constexpr uint64_t kInf = ~0ull;

size_t warp_tier_smem() { return (size_t)(kWarpTierThreads / 32) * 2 * kWarpSlots * 4; }
size_t cta_tier_smem() { return ((size_t)2 * kCtaSlots + kCtaTierThreads + 40) * 4; }
size_t hist_smem() { return (size_t)kBins * 12; }
size_t fd_smem() { return ((size_t)(kFdThreads / 32) * 2 * kFdWarpSlots + 2 * kCtaSlots + kFdThreads) * 4; }

void set_attrs_once() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_agg_warp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_tier_smem());
    cudaFuncSetAttribute(k_agg_cta<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cta_tier_smem());
    cudaFuncSetAttribute(k_agg_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cta_tier_smem());
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
  Counters& readback(Counters* dc) {
    CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return *hc;
  }
  cudaStream_t st;
  int nsm = 148;
  Counters* hc = nullptr;

 private:
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
  k_validate_csr<<<r.nsm * 4, 256, 0, r.st>>>(g.nU, g.m, g.offU, g.adjU, g.nV, bad);
  k_validate_csr<<<r.nsm * 4, 256, 0, r.st>>>(g.nV, g.m, g.offV, g.adjV, g.nU, bad);
  LAUNCHED("k_validate_csr");
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
  uint32_t *slot_cnt, *slot_touch, *slot_dup;
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
  S.nslots = choose_slots(r, g.nU);
  S.slot_cnt = r.alloc<uint32_t>((size_t)S.nslots * g.nU);
  S.slot_touch = r.alloc<uint32_t>((size_t)S.nslots * g.nU);
  S.slot_dup = r.alloc<uint32_t>((size_t)S.nslots * g.nU);
  CK(cudaMemsetAsync(S.slot_cnt, 0, (size_t)S.nslots * g.nU * 4, r.st));
  CK(cudaMemsetAsync(S.vflag, 0, (size_t)std::max<uint32_t>(g.nV, 1) * 4, r.st));
  CK(cudaMemsetAsync(S.c, 0, sizeof(Counters), r.st));
  CK(cudaMemsetAsync(S.sum_d2, 0, 8, r.st));
  if (need_live && g.m) CK(cudaMemcpyAsync(S.adjL, g.adjV, g.m * 4, cudaMemcpyDeviceToDevice, r.st));
  k_init_v<<<r.nsm * 4, 256, 0, r.st>>>(g.nV, g.offV, S.ld, S.sum_d2);
  LAUNCHED("k_init_v");
  k_init_u<<<r.nsm * 8, 256, 0, r.st>>>(g.nU, g.offU, g.adjU, g.offV, S.wc, S.part);
  LAUNCHED("k_init_u");
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
  a.slot_cnt = S.slot_cnt;
  a.slot_touch = S.slot_touch;
  a.slot_dup = S.slot_dup;
  a.nU = S.g.nU;
  a.c = S.c;
  return a;
}

template <int MODE>
void launch_agg(Run& r, const State& S) {
  k_agg_warp<MODE><<<r.nsm * 3, kWarpTierThreads, warp_tier_smem(), r.st>>>(agg_args(S, 0));
  LAUNCHED("k_agg_warp");
  k_agg_cta<MODE><<<r.nsm, kCtaTierThreads, cta_tier_smem(), r.st>>>(agg_args(S, 1));
  LAUNCHED("k_agg_cta");
  k_agg_heavy<MODE><<<S.nslots, kHeavyThreads, 0, r.st>>>(agg_args(S, 2));
  LAUNCHED("k_agg_heavy");
}

void reset_tiers(Run& r, State& S) {
  CK(cudaMemsetAsync(&S.c->ntier[0], 0, 3 * sizeof(uint32_t), r.st));
}

// Butterfly count of every unassigned u (initial count, and §5.1 re-count).
void count_live(Run& r, State& S) {
  reset_tiers(r, S);
  k_classify<0><<<r.nsm * 8, 256, 0, r.st>>>(S.g.nU, nullptr, nullptr, S.g.offU, S.g.adjU, S.ld, S.part,
                                               S.support, S.tier[0], S.tier[1], S.tier[2], nullptr, 0, nullptr,
                                               S.c);
  LAUNCHED("k_classify<count>");
  launch_agg<0>(r, S);
}

void compact(Run& r, State& S) {
  const uint32_t big = 4096;
  k_compact<<<r.nsm * 8, 256, 0, r.st>>>(S.touched, &S.c->ntouched, S.g.offV, S.adjL, S.tmp, S.ld, S.part, big,
                                         S.c);
  LAUNCHED("k_compact");
  k_compact_big<<<r.nsm, 512, 0, r.st>>>(S.touched, &S.c->ntouched, S.g.offV, S.adjL, S.tmp, S.ld, S.part, big,
                                         S.c);
  LAUNCHED("k_compact_big");
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
    k_range_hist<<<r.nsm, 1024, hist_smem(), r.st>>>(nU, S.part, S.support, S.wc, S.init, S.hist_w, S.hist_n,
                                                     S.c);
    LAUNCHED("k_range_hist");
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
      k_select<<<r.nsm * 8, 256, 0, r.st>>>(nU, S.part, S.support, S.wc, bound, pid, S.F, S.c);
      LAUNCHED("k_select");
      k_classify<1><<<r.nsm * 8, 256, 0, r.st>>>(nU, S.F, &S.c->nF, S.g.offU, S.g.adjU, S.ld, S.part, S.support,
                                                   S.tier[0], S.tier[1], S.tier[2], S.vflag, epoch, S.touched,
                                                   S.c);
      LAUNCHED("k_classify<peel>");
      const Counters hc = r.readback(S.c);
      if (hc.nF == 0) break;
      st.rho_cd_iters++;
      if (first) first_wc = hc.sel_wc;
      first = false;
      part_wc += hc.sel_wc;
      if (bound == kInf) {
        // every live vertex is in this batch: nobody is left to update
        if (del) compact(r, S);
        continue;
      }
      const unsigned long long recount_cost = sum_d2 - hc.ld2_drop;  // one-sided re-count cost (g10)
      const bool recount = !(opts & PBNG_OPT_NO_RECOUNT) &&
                           ((opts & PBNG_OPT_FORCE_RECOUNT) || hc.wedges > recount_cost);
      if (recount) {
        // §5.1: re-compute supports of all remaining vertices
        if (del) compact(r, S);
        count_live(r, S);
        st.recounts++;
      } else {
        launch_agg<1>(r, S);
        if (del) compact(r, S);
      }
    }
    if (!del) compact(r, S);
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
  uint8_t* peeled = r.alloc<uint8_t>(nU);
  uint64_t* seg = r.alloc<uint64_t>(S.g.m);
  unsigned long long* fdc = r.alloc<unsigned long long>(3);  // wedges, updates, rounds|ticket
  uint32_t* misc = r.alloc<uint32_t>(2);                     // ticket, rounds_max
  CK(cudaMemsetAsync(pcount, 0, (size_t)np * 4, r.st));
  CK(cudaMemsetAsync(pcur, 0, (size_t)np * 4, r.st));
  CK(cudaMemsetAsync(work, 0, (size_t)np * 8, r.st));
  CK(cudaMemsetAsync(peeled, 0, nU, r.st));
  CK(cudaMemsetAsync(fdc, 0, 24, r.st));
  CK(cudaMemsetAsync(misc, 0, 8, r.st));
  k_part_count<<<r.nsm * 4, 256, np * 4, r.st>>>(nU, S.part, np, pcount);
  LAUNCHED("k_part_count");
  std::vector<uint32_t> hcount(np), hoff(np + 1);
  CK(cudaMemcpyAsync(hcount.data(), pcount, (size_t)np * 4, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  hoff[0] = 0;
  for (uint32_t i = 0; i < np; i++) hoff[i + 1] = hoff[i] + hcount[i];
  CK(cudaMemcpyAsync(poff, hoff.data(), (size_t)(np + 1) * 4, cudaMemcpyHostToDevice, r.st));
  k_part_scatter<<<r.nsm * 8, 256, 0, r.st>>>(nU, S.part, poff, pcur, members);
  LAUNCHED("k_part_scatter");
  k_fd_seg<<<r.nsm * 8, 256, np * 8, r.st>>>(nU, S.g.offU, S.g.adjU, S.g.offV, S.adjL, S.part, np, seg, work);
  LAUNCHED("k_fd_seg");
  std::vector<unsigned long long> hwork(np);
  CK(cudaMemcpyAsync(hwork.data(), work, (size_t)np * 8, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
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
  a.peeled = peeled;
  a.theta = theta;
  a.slot_cnt = S.slot_cnt;
  a.slot_touch = S.slot_touch;
  a.slot_dup = S.slot_dup;
  a.wedges = fdc;
  a.updates = fdc + 1;
  a.rounds_max = misc + 1;
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>({np, (uint32_t)r.nsm, S.nslots}));
  k_fd<<<grid, kFdThreads, fd_smem(), r.st>>>(a);
  LAUNCHED("k_fd");
  cudaEvent_t e2 = r.event();
  unsigned long long hf[3];
  uint32_t hm[2];
  CK(cudaMemcpyAsync(hf, fdc, 24, cudaMemcpyDeviceToHost, r.st));
  CK(cudaMemcpyAsync(hm, misc, 8, cudaMemcpyDeviceToHost, r.st));
  CK(cudaStreamSynchronize(r.st));
  st.wedges_fd = hf[0];
  st.support_updates += hf[1];
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
