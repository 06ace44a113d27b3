/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.c for the rules).
 *
 * Exactness certificate for candidate tip numbers theta' of the peel side U,
 * for graphs where sequential bottom-up peeling (oracle_bup_tip) is too slow
 * ("Exactness certificate"; derived from Definition 2 of the
 * paper, and the bottom-up peeling order).
 *
 *   H_k = { u : theta'_u >= k },  L_k = { u : theta'_u == k }.
 *
 *   (A) for every u:  s_ge(u) = sum_{u' != u, theta'_u' >= theta'_u} C(w(u,u'),2)
 *       >= theta'_u.  Then every H_k is a subgraph in which each vertex lies
 *       in >= k butterflies, so theta_u >= theta'_u (Definition 2).
 *   (C) for every level k: starting from s(u) = butterflies of u inside H_k,
 *       the vertices of L_k can be removed one at a time, each with current
 *       support <= k at its removal (supports drop as L_k vertices leave;
 *       removals only lower supports, so a worklist finds such an order
 *       whenever one exists).
 *       Then the sequence "all of L_0, then L_1, ..." is a valid bottom-up
 *       peeling order in which every vertex of L_k leaves at level <= k, so
 *       theta_u <= theta'_u.
 *   (A) and (C) together give theta' = theta.
 *
 * Functions (OpenMP over vertices / levels; one dense counter array per thread,
 * the paper's private wedge array):
 *   oracle_cert_support_ge  s_ge(u) for a list of u (all u when us == NULL)
 *   oracle_cert_levels      check (C) for a list of levels; returns the number
 *                           of failing levels and the first failing level.
 *
 * Pinned in tests/test_oracle.py: accepts the Definition-2 tip numbers of
 * brute.py on random tiny graphs and rejects every +-1 mutation.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t c2(uint64_t w) { return w * (w - 1) / 2; }

int oracle_cert_support_ge(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                           const uint64_t* offV, const uint32_t* adjV, const uint64_t* theta,
                           const uint32_t* us, uint64_t nus, uint64_t* out) {
  (void)nV;
  const uint64_t n = us ? nus : nU;
  int err = 0;
#pragma omp parallel
  {
    uint32_t* cnt = (uint32_t*)calloc(nU ? nU : 1, sizeof(uint32_t));
    uint32_t* touched = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
    const int mine_ok = cnt && touched;
    if (!mine_ok) {
#pragma omp atomic write
      err = 1;
    }
    {
#pragma omp for schedule(dynamic, 64)
      for (uint64_t i = 0; i < n; i++) {
        if (!mine_ok) continue;
        const uint32_t u = us ? us[i] : (uint32_t)i;
        const uint64_t tu = theta[u];
        uint64_t nt = 0;
        for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
          const uint32_t v = adjU[e];
          for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
            const uint32_t x = adjV[f];
            if (x == u || theta[x] < tu) continue;
            if (cnt[x]++ == 0) touched[nt++] = x;
          }
        }
        uint64_t s = 0;
        for (uint64_t t = 0; t < nt; t++) {
          s += c2(cnt[touched[t]]);
          cnt[touched[t]] = 0;
        }
        out[i] = s;
      }
    }
    free(cnt);
    free(touched);
  }
  return err ? -1 : 0;
}

/* (C) for one level k, members = L_k (sorted or not), m = |L_k|.
 * pos[u] (scratch, all ~0 on entry and exit) indexes members. */
static int check_level(const uint64_t* offU, const uint32_t* adjU, const uint64_t* offV, const uint32_t* adjV,
                       const uint64_t* theta, uint64_t k, const uint32_t* members, uint64_t m, uint32_t* cnt,
                       uint32_t* touched, uint32_t* pos, uint64_t* s, unsigned char* gone, uint32_t* queue) {
  for (uint64_t i = 0; i < m; i++) {
    pos[members[i]] = (uint32_t)i;
    gone[i] = 0;
  }
  /* s(u) = butterflies of u inside H_k */
  for (uint64_t i = 0; i < m; i++) {
    const uint32_t u = members[i];
    uint64_t nt = 0;
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      const uint32_t v = adjU[e];
      for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
        const uint32_t x = adjV[f];
        if (x == u || theta[x] < k) continue;
        if (cnt[x]++ == 0) touched[nt++] = x;
      }
    }
    uint64_t acc = 0;
    for (uint64_t t = 0; t < nt; t++) {
      acc += c2(cnt[touched[t]]);
      cnt[touched[t]] = 0;
    }
    s[i] = acc;
  }
  /* remove L_k one vertex at a time while some remaining vertex has support <= k;
   * removals only lower supports, so the order among removable vertices does
   * not matter (worklist).  gone: 1 = queued, 2 = removed. */
  uint64_t qh = 0, qt = 0, removed = 0;
  for (uint64_t i = 0; i < m; i++)
    if (s[i] <= k) {
      gone[i] = 1;
      queue[qt++] = (uint32_t)i;
    }
  while (qh < qt) {
    const uint64_t b = queue[qh++];
    gone[b] = 2;
    removed++;
    const uint32_t u = members[b];
    uint64_t nt = 0;
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      const uint32_t v = adjU[e];
      for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
        const uint32_t x = adjV[f];
        if (x == u || theta[x] != k || gone[pos[x]] == 2) continue;
        if (cnt[x]++ == 0) touched[nt++] = x;
      }
    }
    for (uint64_t t = 0; t < nt; t++) {
      const uint32_t x = touched[t];
      const uint32_t i = pos[x];
      s[i] -= c2(cnt[x]);
      cnt[x] = 0;
      if (!gone[i] && s[i] <= k) {
        gone[i] = 1;
        queue[qt++] = i;
      }
    }
  }
  const int ok = removed == m;
  for (uint64_t i = 0; i < m; i++) pos[members[i]] = 0xFFFFFFFFu;
  return ok;
}

/* Check (C) for levels[0..nlev): level_members is the concatenation of the
 * member lists, level_off[j]..level_off[j+1] the members of levels[j].
 * Returns the number of failing levels (or -1 on allocation failure);
 * *first_bad = index j of the first failing level (nlev if none). */
int64_t oracle_cert_levels(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                           const uint64_t* offV, const uint32_t* adjV, const uint64_t* theta,
                           const uint64_t* levels, const uint64_t* level_off, const uint32_t* level_members,
                           uint64_t nlev, uint64_t* first_bad) {
  (void)nV;
  int64_t bad = 0;
  uint64_t first = nlev;
  int err = 0;
  uint64_t maxm = 0;
  for (uint64_t j = 0; j < nlev; j++)
    if (level_off[j + 1] - level_off[j] > maxm) maxm = level_off[j + 1] - level_off[j];
#pragma omp parallel
  {
    uint32_t* cnt = (uint32_t*)calloc(nU ? nU : 1, sizeof(uint32_t));
    uint32_t* touched = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
    uint32_t* pos = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
    uint64_t* s = (uint64_t*)malloc((maxm ? maxm : 1) * sizeof(uint64_t));
    unsigned char* gone = (unsigned char*)malloc(maxm ? maxm : 1);
    uint32_t* queue = (uint32_t*)malloc((maxm ? maxm : 1) * sizeof(uint32_t));
    const int mine_ok = cnt && touched && pos && s && gone && queue;
    if (!mine_ok) {
#pragma omp atomic write
      err = 1;
    } else {
      memset(pos, 0xFF, (nU ? nU : 1) * sizeof(uint32_t));
    }
    {
#pragma omp for schedule(dynamic, 1)
      for (uint64_t j = 0; j < nlev; j++) {
        if (!mine_ok) continue;
        const uint64_t m = level_off[j + 1] - level_off[j];
        if (!check_level(offU, adjU, offV, adjV, theta, levels[j], level_members + level_off[j], m, cnt, touched,
                         pos, s, gone, queue)) {
#pragma omp critical
          {
            bad++;
            if (j < first) first = j;
          }
        }
      }
    }
    free(cnt);
    free(touched);
    free(pos);
    free(s);
    free(gone);
    free(queue);
  }
  *first_bad = first;
  return err ? -1 : bad;
}

/* ------------------------------------------------------------------------
 * Certificate for large graphs in ONE wedge pass (config 5: the per-vertex
 * functions above would read every wedge three to four times).
 *
 * Same (A) and (C) as above, and the same butterfly counts as oracle_count,
 * computed over each UNORDERED pair {u, x} once:
 *   key(u) = (theta'_u, u); every list N_v is copied and sorted by key,
 *   descending.  For each u and v in N_u the entries of N_v before u itself
 *   are exactly the partners x with key(x) > key(u), so walking N_v up to u
 *   visits every pair once, from its smaller-key end.  With w = |N_u ∩ N_x|
 *   and c = C(w,2):
 *     support[u] += c, support[x] += c           (every pair: full counts,
 *                                                 Table 1 P:353 / oracle_count)
 *     s_ge[u]    += c                            (theta'_x >= theta'_u always)
 *     s_ge[x]    += c  only if theta'_x == theta'_u
 *   so s_ge is oracle_cert_support_ge's (A) sum for every u.
 * (C) for level k starts from s(u) = s_ge(u) (butterflies of u inside
 * H_k = {theta' >= k}, the same quantity), and a removal walks, for each
 * v in N_u, only the run of N_v whose theta' equals k (contiguous in the
 * sorted copy): the induced subgraph of L_k and all of V, which is all that
 * check_level's filter `theta[x] == k` keeps.
 * Pinned in tests/test_oracle.py against oracle_count, oracle_cert_support_ge
 * and the per-level checker on random graphs (equal outputs, equal verdicts).
 * ------------------------------------------------------------------------ */

static const uint64_t* g_sort_theta;  /* comparator context (set before the parallel sort) */
static int key_desc(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  const uint64_t tx = g_sort_theta[x], ty = g_sort_theta[y];
  if (tx != ty) return tx > ty ? -1 : 1;
  return x > y ? -1 : (x < y ? 1 : 0);
}

/* adjS[offV[v] .. offV[v+1]) = N_v sorted by key descending */
int oracle_cert_sort_lists(uint32_t nV, const uint64_t* offV, const uint32_t* adjV, const uint64_t* theta,
                           uint32_t* adjS) {
  g_sort_theta = theta;
#pragma omp parallel for schedule(dynamic, 256)
  for (uint64_t v = 0; v < nV; v++) {
    const uint64_t a = offV[v], b = offV[v + 1];
    memcpy(adjS + a, adjV + a, (b - a) * sizeof(uint32_t));
    qsort(adjS + a, b - a, sizeof(uint32_t), key_desc);
  }
  return 0;
}

static inline void add_u64(uint64_t* p, uint64_t c) { __atomic_fetch_add(p, c, __ATOMIC_RELAXED); }

/* support[u] (full butterfly counts) and s_ge[u] (certificate (A) sums) for
 * every u, one pass over unordered pairs; adjS from oracle_cert_sort_lists.
 * Both outputs are zeroed here.  *progress (optional) counts finished u. */
int oracle_cert_pass(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU, const uint64_t* offV,
                     const uint32_t* adjS, const uint64_t* theta, uint64_t* support, uint64_t* s_ge,
                     uint64_t* progress) {
  (void)nV;
  int err = 0;
  memset(support, 0, (size_t)nU * sizeof(uint64_t));
  memset(s_ge, 0, (size_t)nU * sizeof(uint64_t));
#pragma omp parallel
  {
    uint32_t* cnt = (uint32_t*)calloc(nU ? nU : 1, sizeof(uint32_t));
    uint32_t* touched = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
    const int mine_ok = cnt && touched;
    if (!mine_ok) {
#pragma omp atomic write
      err = 1;
    }
#pragma omp for schedule(dynamic, 64)
    for (uint64_t i = 0; i < nU; i++) {
      if (!mine_ok) continue;
      const uint32_t u = (uint32_t)i;
      uint64_t nt = 0;
      for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
        const uint32_t v = adjU[e];
        for (uint64_t f = offV[v]; f < offV[v + 1]; f++) {
          const uint32_t x = adjS[f];
          if (x == u) break; /* the rest of N_v has smaller keys */
          if (cnt[x]++ == 0) touched[nt++] = x;
        }
      }
      uint64_t su = 0;
      for (uint64_t t = 0; t < nt; t++) {
        const uint32_t x = touched[t];
        const uint64_t c = c2(cnt[x]);
        cnt[x] = 0;
        if (!c) continue;
        su += c;
        add_u64(&support[x], c);
        if (theta[x] == theta[u]) add_u64(&s_ge[x], c);
      }
      add_u64(&support[u], su);
      add_u64(&s_ge[u], su);
      if (progress) add_u64(progress, 1);
    }
    free(cnt);
    free(touched);
  }
  return err ? -1 : 0;
}

/* first index f in [a, b) of the key-descending list with theta[adjS[f]] <= k */
static uint64_t run_lo(const uint32_t* adjS, const uint64_t* theta, uint64_t a, uint64_t b, uint64_t k) {
  while (a < b) {
    const uint64_t m = a + (b - a) / 2;
    if (theta[adjS[m]] > k) a = m + 1; else b = m;
  }
  return a;
}

/* (C) for one level with the induced runs; s[i] = s_ge of members[i] on entry */
static int check_level_induced(const uint64_t* offU, const uint32_t* adjU, const uint64_t* offV,
                               const uint32_t* adjS, const uint64_t* theta, uint64_t k, const uint32_t* members,
                               uint64_t m, uint32_t* cnt, uint32_t* touched, uint32_t* pos, uint64_t* s,
                               unsigned char* gone, uint32_t* queue) {
  for (uint64_t i = 0; i < m; i++) {
    pos[members[i]] = (uint32_t)i;
    gone[i] = 0;
  }
  uint64_t qh = 0, qt = 0, removed = 0;
  for (uint64_t i = 0; i < m; i++)
    if (s[i] <= k) {
      gone[i] = 1;
      queue[qt++] = (uint32_t)i;
    }
  while (qh < qt) {
    const uint64_t b = queue[qh++];
    gone[b] = 2;
    removed++;
    const uint32_t u = members[b];
    uint64_t nt = 0;
    for (uint64_t e = offU[u]; e < offU[u + 1]; e++) {
      const uint32_t v = adjU[e];
      const uint64_t lo = run_lo(adjS, theta, offV[v], offV[v + 1], k);
      for (uint64_t f = lo; f < offV[v + 1]; f++) {
        const uint32_t x = adjS[f];
        if (theta[x] != k) break; /* end of the level-k run */
        if (x == u || gone[pos[x]] == 2) continue;
        if (cnt[x]++ == 0) touched[nt++] = x;
      }
    }
    for (uint64_t t = 0; t < nt; t++) {
      const uint32_t x = touched[t];
      const uint32_t i = pos[x];
      s[i] -= c2(cnt[x]);
      cnt[x] = 0;
      if (!gone[i] && s[i] <= k) {
        gone[i] = 1;
        queue[qt++] = i;
      }
    }
  }
  const int ok = removed == m;
  for (uint64_t i = 0; i < m; i++) pos[members[i]] = 0xFFFFFFFFu;
  return ok;
}

/* Check (C) for levels[0..nlev) (level_off / level_members as in
 * oracle_cert_levels) from s_ge of oracle_cert_pass.  Returns the number of
 * failing levels (-1 on allocation failure); *first_bad as above. */
int64_t oracle_cert_levels_induced(uint32_t nU, uint32_t nV, const uint64_t* offU, const uint32_t* adjU,
                                   const uint64_t* offV, const uint32_t* adjS, const uint64_t* theta,
                                   const uint64_t* s_ge, const uint64_t* levels, const uint64_t* level_off,
                                   const uint32_t* level_members, uint64_t nlev, uint64_t* first_bad) {
  (void)nV;
  int64_t bad = 0;
  uint64_t first = nlev;
  int err = 0;
  uint64_t maxm = 0;
  for (uint64_t j = 0; j < nlev; j++)
    if (level_off[j + 1] - level_off[j] > maxm) maxm = level_off[j + 1] - level_off[j];
#pragma omp parallel
  {
    uint32_t* cnt = (uint32_t*)calloc(nU ? nU : 1, sizeof(uint32_t));
    uint32_t* touched = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
    uint32_t* pos = (uint32_t*)malloc((nU ? nU : 1) * sizeof(uint32_t));
    uint64_t* s = (uint64_t*)malloc((maxm ? maxm : 1) * sizeof(uint64_t));
    unsigned char* gone = (unsigned char*)malloc(maxm ? maxm : 1);
    uint32_t* queue = (uint32_t*)malloc((maxm ? maxm : 1) * sizeof(uint32_t));
    const int mine_ok = cnt && touched && pos && s && gone && queue;
    if (!mine_ok) {
#pragma omp atomic write
      err = 1;
    } else {
      memset(pos, 0xFF, (nU ? nU : 1) * sizeof(uint32_t));
    }
#pragma omp for schedule(dynamic, 1)
    for (uint64_t j = 0; j < nlev; j++) {
      if (!mine_ok) continue;
      const uint64_t m = level_off[j + 1] - level_off[j];
      const uint32_t* mem = level_members + level_off[j];
      for (uint64_t i = 0; i < m; i++) s[i] = s_ge[mem[i]];
      if (!check_level_induced(offU, adjU, offV, adjS, theta, levels[j], mem, m, cnt, touched, pos, s, gone,
                               queue)) {
#pragma omp critical
        {
          bad++;
          if (j < first) first = j;
        }
      }
    }
    free(cnt);
    free(touched);
    free(pos);
    free(s);
    free(gone);
    free(queue);
  }
  *first_bad = first;
  return err ? -1 : bad;
}
