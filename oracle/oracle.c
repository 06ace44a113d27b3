/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU reference for PBNG tip decomposition
 * (Lakhotia, Kannan, Prasanna, arXiv 2110.12511).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or helper with the
 * CUDA path (paper_2110_12511_b200/); the two meet only in the seeded inputs
 * of graphgen/.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n.
 *
 * Functions
 *   oracle_count     per-vertex butterfly support of every u in U, by plain
 *                    wedge traversal u -> v -> u' and C(w,2) per endpoint pair
 *                    ("combine wedges with common end points",
 *                    Alg.1 l.17-19 P:417-419 C(wedge_count,2) per endpoint).
 *   oracle_bup_tip   sequential bottom-up tip peeling (Alg.2
 *                    P:508-531 specialised to vertices of U as P:493-498
 *                    describes; update rule max(theta, s - C(w,2)) from
 *                    Alg.2 l.11 P:526 / S:259; tie-break lowest id, reading g2).
 *   oracle_count_subset  oracle_count restricted to a list of u (for sampled
 *                    checks at sizes where the full oracle is too slow).
 *   oracle_edge_count per-edge butterfly count (notation table P:353-354,
 *                    Alg.1 per-edge output P:398) by its plain
 *                    definition: sum over u' in N_v \ {u} of (w(u,u') - 1).
 *   oracle_bup_wing  wing decomposition by sequential bottom-up peeling of
 *                    edges, Alg.2 as written, wing numbers per
 *                    U-CSR position.
 *   oracle_tip_level one level of the k-tip hierarchy from tip numbers
 *                    (k-tip = Def. 2): members
 *                    U_k = {theta >= k}, V(H) = V; two members are adjacent
 *                    when they share a butterfly (|N_u ∩ N_u'| >= 2); the
 *                    k-tips are the connected components of that relation
 *                    ("connected by a series of butterflies"), found by
 *                    breadth-first search; label = smallest member id.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): brute-force 4-tuple enumeration,
 * K_{a,b} closed form, sum_U = sum_V identity, tip numbers by Definition 2
 * on tiny graphs, hand-checked golden graphs.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t wedges;   /* (u, v, u') adjacency entries read, u' = u included (g11) */
  uint64_t updates;  /* support decrements applied */
  uint64_t peeled;   /* vertices peeled */
} oracle_stats;

static uint64_t choose2(uint64_t w) { return w * (w - 1) / 2; }

/* support[u] = sum_{u' != u} C(|N_u ∩ N_u'|, 2)  for every u listed in `us`
 * (or all u when us == NULL).  Aggregation with a dense per-vertex counter
 * array and a touched list (the paper's private n-element wedge_count array,
 * P:388-390). */
int oracle_count_subset(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                        const uint64_t* offV, const uint32_t* adjV, const uint32_t* us,
                        uint64_t nus, uint64_t* support, oracle_stats* st) {
  (void)nV;
  uint32_t* cnt = (uint32_t*)calloc(nU ? nU : 1, sizeof(uint32_t));
  uint32_t* touched = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
  if (!cnt || !touched) { free(cnt); free(touched); return -1; }
  uint64_t wedges = 0;
  uint64_t n = us ? nus : nU;
  for (uint64_t i = 0; i < n; i++) {
    uint32_t u = us ? us[i] : (uint32_t)i;
    uint64_t nt = 0;
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      uint32_t v = adjU[e];
      for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
        uint32_t u2 = adjV[f];
        wedges++;
        if (u2 == u) continue;
        if (cnt[u2]++ == 0) touched[nt++] = u2;
      }
    }
    uint64_t s = 0;
    for (uint64_t t = 0; t < nt; t++) {
      s += choose2(cnt[touched[t]]);
      cnt[touched[t]] = 0;
    }
    support[us ? i : u] = s;
  }
  if (st) st->wedges += wedges;
  free(cnt);
  free(touched);
  return 0;
}

int oracle_count(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                 const uint64_t* offV, const uint32_t* adjV, uint64_t* support, oracle_stats* st) {
  return oracle_count_subset(nU, nV, offU, adjU, offV, adjV, NULL, 0, support, st);
}

/* Per-edge butterfly count (notation table: "no. of butterflies in G
 * that contain edge e"; the per-edge output of Alg.1).
 * The plain definition written out: a butterfly through e = (u, v) is a pair
 * (u', v') with u' != u, v' != v and edges (u, v'), (u', v), (u', v'); for a
 * fixed u' in N_v \ {u} the admissible v' are N_u ∩ N_u' \ {v}, of which
 * there are w(u,u') - 1 (v itself is common).  So
 *     edge_support[e] = sum_{u' in N_v, u' != u} (w(u,u') - 1),
 * w from the same dense counters as oracle_count.  edge_support is indexed by
 * the position e of the edge in the U-side CSR (offU/adjU). */
int oracle_edge_count(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                      const uint64_t* offV, const uint32_t* adjV, uint64_t* edge_support, oracle_stats* st) {
  (void)nV;
  uint32_t* cnt = (uint32_t*)calloc(nU ? nU : 1, sizeof(uint32_t));
  uint32_t* touched = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
  if (!cnt || !touched) { free(cnt); free(touched); return -1; }
  uint64_t wedges = 0;
  for (uint32_t u = 0; u < nU; u++) {
    uint64_t nt = 0;
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      uint32_t v = adjU[e];
      for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
        uint32_t u2 = adjV[f];
        wedges++;
        if (u2 == u) continue;
        if (cnt[u2]++ == 0) touched[nt++] = u2;
      }
    }
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      uint32_t v = adjU[e];
      uint64_t s = 0;
      for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
        uint32_t u2 = adjV[f];
        if (u2 == u) continue;
        s += cnt[u2] - 1;
      }
      edge_support[e] = s;
    }
    for (uint64_t t = 0; t < nt; t++) cnt[touched[t]] = 0;
  }
  if (st) st->wedges += 2 * wedges;
  free(cnt);
  free(touched);
  return 0;
}

/* ---- indexed binary min-heap keyed by (support, id) --------------------- */
typedef struct {
  uint32_t* heap;   /* heap[i] = vertex id */
  uint32_t* pos;    /* pos[u] = index in heap, or UINT32_MAX when popped */
  const uint64_t* key;
  uint32_t size;
} iheap;

static int less_(const iheap* h, uint32_t a, uint32_t b) {
  return h->key[a] < h->key[b] || (h->key[a] == h->key[b] && a < b);
}
static void swap_(iheap* h, uint32_t i, uint32_t j) {
  uint32_t a = h->heap[i], b = h->heap[j];
  h->heap[i] = b; h->heap[j] = a;
  h->pos[b] = i; h->pos[a] = j;
}
static void up_(iheap* h, uint32_t i) {
  while (i > 0) {
    uint32_t p = (i - 1) / 2;
    if (!less_(h, h->heap[i], h->heap[p])) break;
    swap_(h, i, p);
    i = p;
  }
}
static void down_(iheap* h, uint32_t i) {
  for (;;) {
    uint32_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->size && less_(h, h->heap[l], h->heap[m])) m = l;
    if (r < h->size && less_(h, h->heap[r], h->heap[m])) m = r;
    if (m == i) break;
    swap_(h, i, m);
    i = m;
  }
}
static uint32_t pop_(iheap* h) {
  uint32_t top = h->heap[0];
  h->size--;
  if (h->size) {
    h->heap[0] = h->heap[h->size];
    h->pos[h->heap[0]] = 0;
    down_(h, 0);
  }
  h->pos[top] = UINT32_MAX;
  return top;
}

/* Sequential bottom-up peeling of U (tip decomposition).
 *   support <- per-vertex butterfly counts            (Alg.2 l.1)
 *   while U non-empty:                                 (Alg.2 l.2)
 *     u <- argmin support (lowest id among ties)       (Alg.2 l.3, g2)
 *     theta_u <- support_u; remove u                   (Alg.2 l.4)
 *     for every remaining u' sharing w = |N_u ∩ N_u'| >= 2 common neighbours:
 *       support_u' <- max(theta_u, support_u' - C(w,2)) (Alg.2 l.11 P:526)
 * Removed vertices are skipped during traversal (equivalent to deleting their
 * edges). */
int oracle_bup_tip(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                   const uint64_t* offV, const uint32_t* adjV, uint64_t* theta, oracle_stats* st) {
  (void)nV;
  if (nU == 0) return 0;
  uint64_t* support = (uint64_t*)malloc(nU * sizeof(uint64_t));
  unsigned char* alive = (unsigned char*)malloc(nU);
  uint32_t* cnt = (uint32_t*)calloc(nU, sizeof(uint32_t));
  uint32_t* touched = (uint32_t*)malloc(nU * sizeof(uint32_t));
  iheap h;
  h.heap = (uint32_t*)malloc(nU * sizeof(uint32_t));
  h.pos = (uint32_t*)malloc(nU * sizeof(uint32_t));
  if (!support || !alive || !cnt || !touched || !h.heap || !h.pos) return -1;
  oracle_stats local = {0, 0, 0};
  if (oracle_count(nU, nV, offU, adjU, offV, adjV, support, &local)) return -1;

  h.key = support;
  h.size = nU;
  for (uint32_t u = 0; u < nU; u++) { h.heap[u] = u; h.pos[u] = u; alive[u] = 1; }
  for (int64_t i = (int64_t)nU / 2 - 1; i >= 0; i--) down_(&h, (uint32_t)i);

  while (h.size) {
    uint32_t u = pop_(&h);
    uint64_t th = support[u];
    theta[u] = th;
    alive[u] = 0;
    local.peeled++;
    uint64_t nt = 0;
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      uint32_t v = adjU[e];
      for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
        uint32_t u2 = adjV[f];
        local.wedges++;
        if (!alive[u2]) continue;
        if (cnt[u2]++ == 0) touched[nt++] = u2;
      }
    }
    for (uint64_t t = 0; t < nt; t++) {
      uint32_t u2 = touched[t];
      uint64_t w = cnt[u2];
      cnt[u2] = 0;
      if (w < 2) continue;
      uint64_t d = choose2(w);
      uint64_t s = support[u2];
      uint64_t ns = (s >= th + d) ? s - d : th; /* max(theta_u, s - d) without wrap */
      local.updates++;
      if (ns != s) {
        support[u2] = ns;
        up_(&h, h.pos[u2]);
      }
    }
  }
  if (st) { st->wedges += local.wedges; st->updates += local.updates; st->peeled += local.peeled; }
  free(support); free(alive); free(cnt); free(touched); free(h.heap); free(h.pos);
  return 0;
}

/* ---- wing decomposition (edges) ------------------------------------------
 * Bottom-up peeling of edges exactly as Alg.2: support = per-edge
 * butterfly counts (l.1, oracle_edge_count), repeatedly peel the edge of
 * minimum support (l.3, tie-break lowest U-CSR position), theta_e = its support
 * (l.4), and for every butterfly (u,v,u',v') of the current graph through
 * e = (u,v) (l.7-10: v' in N_u \ {v}, u' in N_v' \ {u} with (u',v) in E(G))
 * set support <- max(theta_e, support - 1) on e1=(u,v'), e2=(u',v), e3=(u',v')
 * (l.11).  theta is indexed by U-CSR position.  Edge lookup by binary search
 * in sorted copies of the U lists. */
typedef struct { uint32_t v; uint32_t e; } vpos;
static int vpos_cmp(const void* a, const void* b) {
  uint32_t x = ((const vpos*)a)->v, y = ((const vpos*)b)->v;
  return x < y ? -1 : (x > y);
}
static int64_t find_edge(const uint64_t* offU, const vpos* sorted, uint32_t u, uint32_t v) {
  uint64_t lo = offU[u], hi = offU[u + 1];
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (sorted[mid].v < v) lo = mid + 1; else hi = mid;
  }
  return (lo < offU[u + 1] && sorted[lo].v == v) ? (int64_t)sorted[lo].e : -1;
}

int oracle_bup_wing(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                    const uint64_t* offV, const uint32_t* adjV, uint64_t* theta, oracle_stats* st) {
  uint64_t m = offU[nU];
  if (m == 0) return 0;
  if (m >= UINT32_MAX) return -1;
  uint64_t* support = (uint64_t*)malloc(m * sizeof(uint64_t));
  unsigned char* alive = (unsigned char*)malloc(m);
  uint32_t* row = (uint32_t*)malloc(m * sizeof(uint32_t));
  vpos* sorted = (vpos*)malloc(m * sizeof(vpos));
  iheap h;
  h.heap = (uint32_t*)malloc(m * sizeof(uint32_t));
  h.pos = (uint32_t*)malloc(m * sizeof(uint32_t));
  if (!support || !alive || !row || !sorted || !h.heap || !h.pos) return -1;
  oracle_stats local = {0, 0, 0};
  if (oracle_edge_count(nU, nV, offU, adjU, offV, adjV, support, &local)) return -1;
  for (uint32_t u = 0; u < nU; u++) {
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      row[e] = u;
      sorted[e].v = adjU[e];
      sorted[e].e = (uint32_t)e;
    }
    qsort(sorted + offU[u], offU[u + 1] - offU[u], sizeof(vpos), vpos_cmp);
  }
  h.key = support;
  h.size = (uint32_t)m;
  for (uint32_t e = 0; e < m; e++) { h.heap[e] = e; h.pos[e] = e; alive[e] = 1; }
  for (int64_t i = (int64_t)m / 2 - 1; i >= 0; i--) down_(&h, (uint32_t)i);
  while (h.size) {
    uint32_t e = pop_(&h);
    uint64_t th = support[e];
    theta[e] = th;
    alive[e] = 0;
    local.peeled++;
    uint32_t u = row[e], v = adjU[e];
    for (uint64_t e1 = offU[u]; e1 < offU[u + 1]; e1++) {
      if (!alive[e1]) continue;           /* e1 = (u, v') in E(G), v' != v (e is gone) */
      uint32_t v2 = adjU[e1];
      for (uint64_t f = offV[v2]; f < offV[v2 + 1]; f++) {
        uint32_t u2 = adjV[f];
        local.wedges++;
        if (u2 == u) continue;
        int64_t e3 = find_edge(offU, sorted, u2, v2);   /* (u', v') */
        int64_t e2 = find_edge(offU, sorted, u2, v);    /* (u', v)  */
        if (e3 < 0 || e2 < 0 || !alive[e3] || !alive[e2]) continue;
        uint64_t ids[3] = {e1, (uint64_t)e2, (uint64_t)e3};
        for (int j = 0; j < 3; j++) {
          uint64_t x = ids[j], s = support[x];
          uint64_t ns = s > th ? s - 1 : th;  /* max(theta_e, s - 1) */
          local.updates++;
          if (ns != s) { support[x] = ns; up_(&h, h.pos[x]); }
        }
      }
    }
  }
  if (st) { st->wedges += local.wedges; st->updates += local.updates; st->peeled += local.peeled; }
  free(support); free(alive); free(row); free(sorted); free(h.heap); free(h.pos);
  return 0;
}

/* comp[u] = smallest id of u's k-tip if theta[u] >= k, else 0xFFFFFFFF;
 * returns the number of k-tips (or -1 on allocation failure).  Plain BFS over
 * members; the neighbours of a member are the members it shares >= 2
 * neighbours with, found by the same dense counter array as oracle_count.
 * Members are visited in increasing id, so each BFS root is the smallest id
 * of its component. */
int64_t oracle_tip_level(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                         const uint64_t* offV, const uint32_t* adjV, const uint64_t* theta, uint64_t k,
                         uint32_t* comp) {
  (void)nV;
  size_t n1 = nU ? nU : 1;
  uint32_t* cnt = (uint32_t*)calloc(n1, sizeof(uint32_t));
  uint32_t* touched = (uint32_t*)malloc(n1 * sizeof(uint32_t));
  uint32_t* queue = (uint32_t*)malloc(n1 * sizeof(uint32_t));
  if (!cnt || !touched || !queue) { free(cnt); free(touched); free(queue); return -1; }
  for (uint32_t u = 0; u < nU; u++) comp[u] = 0xFFFFFFFFu;
  int64_t ncomp = 0;
  for (uint32_t root = 0; root < nU; root++) {
    if (theta[root] < k || comp[root] != 0xFFFFFFFFu) continue;
    ncomp++;
    uint64_t head = 0, tail = 0;
    comp[root] = root;
    queue[tail++] = root;
    while (head < tail) {
      uint32_t u = queue[head++];
      uint64_t nt = 0;
      for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
        uint32_t v = adjU[e];
        for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
          uint32_t u2 = adjV[f];
          if (u2 == u || theta[u2] < k) continue;
          if (cnt[u2]++ == 0) touched[nt++] = u2;
        }
      }
      for (uint64_t t = 0; t < nt; t++) {
        uint32_t u2 = touched[t];
        if (cnt[u2] >= 2 && comp[u2] == 0xFFFFFFFFu) {
          comp[u2] = root;
          queue[tail++] = u2;
        }
        cnt[u2] = 0;
      }
    }
  }
  free(cnt);
  free(touched);
  free(queue);
  return ncomp;
}
