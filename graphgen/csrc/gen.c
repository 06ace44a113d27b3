/*
 * graphgen — seeded synthetic bipartite graph generator (shared input module).
 *
 * This file holds NO part of the tip-decomposition method: it only draws
 * edges and lays them out as two CSR arrays (U side and V side).  Both the
 * CPU oracle (oracle/) and the CUDA path (paper_2110_12511_b200/) read the
 * bytes it produces; it imports neither of them.
 *
 * Recipe (SURVEY.md §8(d) reading R1):
 *   kind 0  uniform:   u ~ U[0,nU), v ~ U[0,nV) per candidate; keep the first
 *                      m distinct pairs of the candidate stream.
 *   kind 1  blocks:    nblocks complete blocks K_{a,b}, a,b ~ U{bmin..bmax};
 *                      plus ceil(noise_pct% of block edges) distinct noise
 *                      edges (u, v) drawn uniformly with block(u) != block(v).
 *   kind 2  chung-lu:  i.i.d. weights from the continuous power law
 *                      pdf ∝ x^-gamma on [1, cap] (inverse CDF); rescale to the
 *                      mean m/n, cap; repeated 5x.  Endpoints drawn
 *                      independently by Vose alias tables; keep the first m
 *                      distinct pairs.
 * Randomness: counter-based splitmix64 (stream key, index) so every candidate
 * is a pure function of (seed, stream, index): byte-identical output on any
 * host, thread count or run.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct {
  int kind;                 /* 0 uniform, 1 blocks, 2 chung-lu */
  uint32_t nU, nV;          /* side sizes (kinds 0 and 2) */
  uint64_t m;               /* target distinct edges (kinds 0 and 2) */
  double gammaU, gammaV;    /* power-law exponents (kind 2) */
  double capU, capV;        /* max expected degree (kind 2) */
  uint64_t seed;
  uint32_t nblocks, bmin, bmax, noise_pct; /* kind 1 */
} gen_params;

typedef struct {
  uint32_t nU, nV;
  uint64_t m;
  uint64_t* keys;           /* sorted edge keys u*nV+v, length m */
} gen_graph;

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed + 0x632BE59BD9B4E019ULL) ^ (stream * 0xD1B54A32D192ED03ULL));
}
static inline uint64_t rnd(uint64_t key, uint64_t i) {
  return mix64(key + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
static inline uint32_t bounded(uint64_t r, uint32_t n) {
  return (uint32_t)(((r >> 32) * (uint64_t)n) >> 32);
}
static inline double unit(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

/* ---- LSD radix sort of (key, idx) pairs, stable, 11-bit digits ---------- */
static int radix_sort_kv(uint64_t* keys, uint32_t* idx, uint64_t n, uint64_t maxkey) {
  int bits = 0;
  while (bits < 64 && (maxkey >> bits) != 0) bits++;
  if (n < 2 || bits == 0) return 0;
  uint64_t* k2 = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint32_t* i2 = idx ? (uint32_t*)malloc(n * sizeof(uint32_t)) : NULL;
  if (!k2 || (idx && !i2)) { free(k2); free(i2); return -1; }
  uint64_t* cnt = (uint64_t*)malloc(2048 * sizeof(uint64_t));
  uint64_t *ks = keys, *kd = k2;
  uint32_t *is = idx, *id = i2;
  for (int sh = 0; sh < bits; sh += 11) {
    memset(cnt, 0, 2048 * sizeof(uint64_t));
    for (uint64_t j = 0; j < n; j++) cnt[(ks[j] >> sh) & 2047]++;
    uint64_t s = 0;
    for (int b = 0; b < 2048; b++) { uint64_t c = cnt[b]; cnt[b] = s; s += c; }
    for (uint64_t j = 0; j < n; j++) {
      uint64_t p = cnt[(ks[j] >> sh) & 2047]++;
      kd[p] = ks[j];
      if (is) id[p] = is[j];
    }
    uint64_t* tk = ks; ks = kd; kd = tk;
    uint32_t* ti = is; is = id; id = ti;
  }
  if (ks != keys) {
    memcpy(keys, ks, n * sizeof(uint64_t));
    if (idx) memcpy(idx, is, n * sizeof(uint32_t));
  }
  free(cnt);
  free(ks == keys ? kd : ks);
  if (idx) free(is == idx ? id : is);
  return 0;
}

/* ---- alias tables (Vose) ------------------------------------------------ */
typedef struct { uint32_t n; uint64_t* thr; uint32_t* alias; } alias_t;

static int alias_build(alias_t* a, const double* w, uint32_t n) {
  a->n = n;
  a->thr = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  a->alias = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  double* p = (double*)malloc((size_t)n * sizeof(double));
  uint32_t* small = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  uint32_t* large = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  if (!a->thr || !a->alias || !p || !small || !large) return -1;
  double tot = 0;
  for (uint32_t i = 0; i < n; i++) tot += w[i];
  uint64_t ns = 0, nl = 0;
  for (uint32_t i = 0; i < n; i++) {
    p[i] = w[i] * (double)n / tot;
    if (p[i] < 1.0) small[ns++] = i; else large[nl++] = i;
  }
  while (ns && nl) {
    uint32_t s = small[--ns], l = large[--nl];
    a->thr[s] = (uint64_t)(p[s] * 4294967296.0);
    a->alias[s] = l;
    p[l] = (p[l] + p[s]) - 1.0;
    if (p[l] < 1.0) small[ns++] = l; else large[nl++] = l;
  }
  while (nl) { uint32_t l = large[--nl]; a->thr[l] = 1ULL << 32; a->alias[l] = l; }
  while (ns) { uint32_t s = small[--ns]; a->thr[s] = 1ULL << 32; a->alias[s] = s; }
  free(p); free(small); free(large);
  return 0;
}
static inline uint32_t alias_draw(const alias_t* a, uint64_t r) {
  uint32_t col = bounded(r, a->n);
  return ((r & 0xFFFFFFFFULL) < a->thr[col]) ? col : a->alias[col];
}
static void alias_free(alias_t* a) { free(a->thr); free(a->alias); }

static double* chung_lu_weights(uint32_t n, uint64_t m, double gamma, double cap, uint64_t key) {
  double* w = (double*)malloc((size_t)n * sizeof(double));
  if (!w) return NULL;
  double e = 1.0 - gamma, top = pow(cap, e) - 1.0;
  for (uint32_t i = 0; i < n; i++) w[i] = pow(1.0 + unit(rnd(key, i)) * top, 1.0 / e);
  double target = (double)m / (double)n;
  for (int it = 0; it < 5; it++) {
    double s = 0;
    for (uint32_t i = 0; i < n; i++) s += w[i];
    double f = target / (s / (double)n);
    for (uint32_t i = 0; i < n; i++) { w[i] *= f; if (w[i] > cap) w[i] = cap; }
  }
  return w;
}

/* ---- first m distinct keys of a candidate stream ------------------------ */
typedef uint64_t (*cand_fn)(const void* ctx, uint64_t j); /* returns key or ctx sentinel */

typedef struct {
  int kind;
  uint32_t nU, nV;
  uint64_t kU, kV;
  const alias_t *aU, *aV;
  const uint32_t *blkU, *blkV; /* block id per vertex (kind 1) */
  uint64_t sentinel;           /* nU*nV: rejected candidate */
} cand_ctx;

static uint64_t cand(const cand_ctx* c, uint64_t j) {
  uint32_t u, v;
  if (c->kind == 2) { u = alias_draw(c->aU, rnd(c->kU, j)); v = alias_draw(c->aV, rnd(c->kV, j)); }
  else { u = bounded(rnd(c->kU, j), c->nU); v = bounded(rnd(c->kV, j), c->nV); }
  if (c->kind == 1 && c->blkU[u] == c->blkV[v]) return c->sentinel;
  return (uint64_t)u * c->nV + v;
}

static uint64_t* first_distinct(const cand_ctx* c, uint64_t m) {
  if (m == 0) return (uint64_t*)malloc(8);
  uint64_t K = m + m / 8 + 1024;
  for (;;) {
    uint64_t* keys = (uint64_t*)malloc(K * sizeof(uint64_t));
    uint32_t* idx = (uint32_t*)malloc(K * sizeof(uint32_t));
    unsigned char* mark = (unsigned char*)calloc(K, 1);
    if (!keys || !idx || !mark || K > 0xFFFFFFFFULL) { free(keys); free(idx); free(mark); return NULL; }
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < (int64_t)K; j++) { keys[j] = cand(c, (uint64_t)j); idx[j] = (uint32_t)j; }
    if (radix_sort_kv(keys, idx, K, c->sentinel)) { free(keys); free(idx); free(mark); return NULL; }
    uint64_t D = 0;
    for (uint64_t j = 0; j < K; j++) {
      if (keys[j] == c->sentinel) break;
      if (j == 0 || keys[j] != keys[j - 1]) { mark[idx[j]] = 1; D++; }
    }
    if (D < m) { free(keys); free(idx); free(mark); K = K + K / 3 + 1024; continue; }
    uint64_t cnt = 0, J = 0;
    for (uint64_t j = 0; j < K; j++) { cnt += mark[j]; if (cnt == m) { J = j; break; } }
    uint64_t* out = (uint64_t*)malloc(m * sizeof(uint64_t));
    uint64_t o = 0;
    for (uint64_t j = 0; j < K && o < m; j++) {
      if (keys[j] == c->sentinel) break;
      if ((j == 0 || keys[j] != keys[j - 1]) && idx[j] <= J) out[o++] = keys[j];
    }
    free(keys); free(idx); free(mark);
    return out;
  }
}

void* gen_build(const gen_params* p) {
  gen_graph* g = (gen_graph*)calloc(1, sizeof(gen_graph));
  if (!g) return NULL;
  cand_ctx c;
  memset(&c, 0, sizeof(c));
  c.kind = p->kind;
  c.kU = stream_key(p->seed, 1);
  c.kV = stream_key(p->seed, 2);
  if (p->kind == 0) {
    g->nU = c.nU = p->nU; g->nV = c.nV = p->nV;
    c.sentinel = (uint64_t)c.nU * c.nV;
    if (p->m > c.sentinel) { free(g); return NULL; }
    g->m = p->m;
    g->keys = first_distinct(&c, p->m);
  } else if (p->kind == 2) {
    g->nU = c.nU = p->nU; g->nV = c.nV = p->nV;
    c.sentinel = (uint64_t)c.nU * c.nV;
    double* wU = chung_lu_weights(p->nU, p->m, p->gammaU, p->capU, stream_key(p->seed, 3));
    double* wV = chung_lu_weights(p->nV, p->m, p->gammaV, p->capV, stream_key(p->seed, 4));
    alias_t aU, aV;
    if (!wU || !wV || alias_build(&aU, wU, p->nU) || alias_build(&aV, wV, p->nV)) { free(g); return NULL; }
    free(wU); free(wV);
    c.aU = &aU; c.aV = &aV;
    g->m = p->m;
    g->keys = first_distinct(&c, p->m);
    alias_free(&aU); alias_free(&aV);
  } else if (p->kind == 1) {
    uint64_t kA = stream_key(p->seed, 5), kB = stream_key(p->seed, 6);
    uint32_t nb = p->nblocks, span = p->bmax - p->bmin + 1;
    uint32_t *a = (uint32_t*)malloc(nb * 4), *b = (uint32_t*)malloc(nb * 4);
    uint64_t nU = 0, nV = 0, eb = 0;
    for (uint32_t k = 0; k < nb; k++) {
      a[k] = p->bmin + bounded(rnd(kA, k), span);
      b[k] = p->bmin + bounded(rnd(kB, k), span);
      nU += a[k]; nV += b[k]; eb += (uint64_t)a[k] * b[k];
    }
    uint32_t* blkU = (uint32_t*)malloc(nU * 4);
    uint32_t* blkV = (uint32_t*)malloc(nV * 4);
    uint64_t ou = 0, ov = 0;
    for (uint32_t k = 0; k < nb; k++) {
      for (uint32_t i = 0; i < a[k]; i++) blkU[ou++] = k;
      for (uint32_t i = 0; i < b[k]; i++) blkV[ov++] = k;
    }
    g->nU = c.nU = (uint32_t)nU; g->nV = c.nV = (uint32_t)nV;
    c.blkU = blkU; c.blkV = blkV;
    c.sentinel = nU * nV;
    uint64_t noise = (eb * p->noise_pct + 99) / 100;
    c.kU = stream_key(p->seed, 7); c.kV = stream_key(p->seed, 8);
    uint64_t* nk = first_distinct(&c, noise);
    g->m = eb + noise;
    g->keys = (uint64_t*)malloc(g->m * sizeof(uint64_t));
    uint64_t o = 0; ou = 0; ov = 0;
    for (uint32_t k = 0; k < nb; k++) {
      for (uint32_t i = 0; i < a[k]; i++)
        for (uint32_t j = 0; j < b[k]; j++) g->keys[o++] = (ou + i) * nV + (ov + j);
      ou += a[k]; ov += b[k];
    }
    memcpy(g->keys + o, nk, noise * sizeof(uint64_t));
    radix_sort_kv(g->keys, NULL, g->m, c.sentinel);
    free(nk); free(a); free(b); free(blkU); free(blkV);
  } else {
    free(g);
    return NULL;
  }
  if (!g->keys) { free(g); return NULL; }
  return g;
}

void gen_info(const void* h, uint32_t* nU, uint32_t* nV, uint64_t* m) {
  const gen_graph* g = (const gen_graph*)h;
  *nU = g->nU; *nV = g->nV; *m = g->m;
}

/* Fill caller buffers: offU[nU+1], adjU[m] (each list ascending in v),
 * offV[nV+1], adjV[m] (each list ascending in u). */
void gen_fill(const void* h, uint64_t* offU, uint32_t* adjU, uint64_t* offV, uint32_t* adjV) {
  const gen_graph* g = (const gen_graph*)h;
  memset(offU, 0, (g->nU + 1ULL) * 8);
  memset(offV, 0, (g->nV + 1ULL) * 8);
  for (uint64_t e = 0; e < g->m; e++) {
    uint64_t k = g->keys[e];
    offU[k / g->nV + 1]++;
    offV[k % g->nV + 1]++;
  }
  for (uint32_t i = 0; i < g->nU; i++) offU[i + 1] += offU[i];
  for (uint32_t i = 0; i < g->nV; i++) offV[i + 1] += offV[i];
  uint64_t* cur = (uint64_t*)malloc(((uint64_t)g->nV + 1) * 8);
  memcpy(cur, offV, ((uint64_t)g->nV + 1) * 8);
  for (uint64_t e = 0; e < g->m; e++) {
    uint64_t k = g->keys[e];
    uint32_t u = (uint32_t)(k / g->nV), v = (uint32_t)(k % g->nV);
    adjU[e] = v;
    adjV[cur[v]++] = u;
  }
  free(cur);
}

void gen_free(void* h) {
  gen_graph* g = (gen_graph*)h;
  if (!g) return;
  free(g->keys);
  free(g);
}
