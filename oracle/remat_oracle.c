/* remat_oracle.c — CPU restatement of the reference recomputation solver.
 *
 * TEST INFRASTRUCTURE ONLY: the parity checker for the CUDA path and the CPU
 * baseline ("port") timed by bench.py.  Never part of the product library.
 *
 * Each function restates the reference Python at the cited file:line of
 * /root/reference/pkg/src/remat (push-style DP with sparse cells realised as
 * dense per-member rows over t in [0, T(V)]).  Parity is pinned against the
 * Python reference's own outputs: the JSON fixtures in tests/golden (made by tests/golden/make_golden.py).
 */
#include "remat_oracle.h"

#include <limits.h>
#include <stdio.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EMPTY INT64_MAX

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* set algebra (graph.py:117-164)                                            */
/* ------------------------------------------------------------------------ */

static int popcount_set(const uint64_t *s, int w) {
  int c = 0;
  for (int k = 0; k < w; k++) c += __builtin_popcountll(s[k]);
  return c;
}

static int64_t weight_of(const int64_t *cost, const uint64_t *s, int w) {
  int64_t acc = 0;
  for (int k = 0; k < w; k++) {
    uint64_t x = s[k];
    while (x) {
      acc += cost[k * 64 + __builtin_ctzll(x)];
      x &= x - 1;
    }
  }
  return acc;
}

static void full_set(int n, int w, uint64_t *out) {
  for (int k = 0; k < w; k++) {
    int lo = k * 64;
    int cnt = n - lo;
    out[k] = cnt >= 64 ? ~0ull : (cnt <= 0 ? 0ull : ((1ull << cnt) - 1));
  }
}

/* delta_plus (graph.py:132-137) */
static void delta_plus(const orc_graph *g, const uint64_t *s, uint64_t *out) {
  int w = g->w;
  memset(out, 0, sizeof(uint64_t) * w);
  for (int k = 0; k < w; k++) {
    uint64_t x = s[k];
    while (x) {
      int v = k * 64 + __builtin_ctzll(x);
      x &= x - 1;
      for (int q = 0; q < w; q++) out[q] |= g->succs[(size_t)v * w + q];
    }
  }
}

/* delta_minus (graph.py:140-145) */
static void delta_minus(const orc_graph *g, const uint64_t *s, uint64_t *out) {
  int w = g->w;
  memset(out, 0, sizeof(uint64_t) * w);
  for (int k = 0; k < w; k++) {
    uint64_t x = s[k];
    while (x) {
      int v = k * 64 + __builtin_ctzll(x);
      x &= x - 1;
      for (int q = 0; q < w; q++) out[q] |= g->preds[(size_t)v * w + q];
    }
  }
}

/* boundary (graph.py:157-164): v in L with a successor outside L */
static void boundary(const orc_graph *g, const uint64_t *lower, uint64_t *out) {
  int w = g->w;
  memset(out, 0, sizeof(uint64_t) * w);
  for (int k = 0; k < w; k++) {
    uint64_t x = lower[k];
    while (x) {
      int b = __builtin_ctzll(x);
      int v = k * 64 + b;
      x &= x - 1;
      const uint64_t *sv = g->succs + (size_t)v * w;
      int outside = 0;
      for (int q = 0; q < w && !outside; q++) outside = (sv[q] & ~lower[q]) != 0;
      if (outside) out[k] |= 1ull << b;
    }
  }
}

static int is_lower_set(const orc_graph *g, const uint64_t *s) {
  int w = g->w;
  uint64_t *dm = malloc(sizeof(uint64_t) * w);
  delta_minus(g, s, dm);
  int ok = 1;
  for (int k = 0; k < w; k++) ok &= (dm[k] & ~s[k]) == 0;
  free(dm);
  return ok;
}

/* ------------------------------------------------------------------------ */
/* families (lattice.py)                                                     */
/* ------------------------------------------------------------------------ */

typedef struct {
  int w;
  int64_t count, capacity;
  uint64_t *masks; /* [capacity][w] */
} maskvec;

static int mv_push(maskvec *v, const uint64_t *m) {
  if (v->count == v->capacity) {
    int64_t nc = v->capacity ? v->capacity * 2 : 1024;
    uint64_t *p = realloc(v->masks, sizeof(uint64_t) * v->w * nc);
    if (!p) return ORC_ERR_NOMEM;
    v->masks = p;
    v->capacity = nc;
  }
  memcpy(v->masks + (size_t)v->count * v->w, m, sizeof(uint64_t) * v->w);
  v->count++;
  return ORC_OK;
}

static int g_sort_w; /* qsort comparator context (oracle is not reentrant) */

/* LowerSetFamily.from_masks order (lattice.py:44-47): (popcount, mask int) */
static int cmp_family(const void *a, const void *b) {
  const uint64_t *x = a, *y = b;
  int w = g_sort_w;
  int px = popcount_set(x, w), py = popcount_set(y, w);
  if (px != py) return px < py ? -1 : 1;
  for (int k = w - 1; k >= 0; k--)
    if (x[k] != y[k]) return x[k] < y[k] ? -1 : 1;
  return 0;
}

static void sort_dedup(maskvec *v) {
  int w = v->w;
  g_sort_w = w;
  qsort(v->masks, v->count, sizeof(uint64_t) * w, cmp_family);
  int64_t out = 0;
  for (int64_t i = 0; i < v->count; i++) {
    if (out > 0 && memcmp(v->masks + (out - 1) * w, v->masks + i * w, 8 * w) == 0) continue;
    if (out != i) memcpy(v->masks + out * w, v->masks + i * w, 8 * w);
    out++;
  }
  v->count = out;
}

/* open-addressing set of masks, used by the DFS enumeration's `seen` */
typedef struct {
  int w;
  int64_t cap;  /* power of two */
  int64_t *slot; /* index into vec or -1 */
} maskset;

static uint64_t hash_mask(const uint64_t *m, int w) {
  uint64_t h = 0x9E3779B97F4A7C15ull;
  for (int k = 0; k < w; k++) {
    h ^= m[k] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xBF58476D1CE4E5B9ull;
  }
  return h ^ (h >> 31);
}

static int ms_grow(maskset *s, const maskvec *v) {
  int64_t nc = s->cap ? s->cap * 2 : 4096;
  int64_t *ns = malloc(sizeof(int64_t) * nc);
  if (!ns) return ORC_ERR_NOMEM;
  for (int64_t i = 0; i < nc; i++) ns[i] = -1;
  for (int64_t i = 0; i < v->count; i++) {
    uint64_t h = hash_mask(v->masks + i * v->w, v->w) & (nc - 1);
    while (ns[h] >= 0) h = (h + 1) & (nc - 1);
    ns[h] = i;
  }
  free(s->slot);
  s->slot = ns;
  s->cap = nc;
  return ORC_OK;
}

/* all_lower_sets (lattice.py:59-84): DFS by single-node extension with a
 * `seen` set; error as soon as more than `cap` sets have been seen. */
static int enumerate_full(const orc_graph *g, int64_t cap, maskvec *out) {
  int n = g->n, w = g->w;
  if (cap < (int64_t)n + 1) return ORC_ERR_ARG;
  maskvec vec = {w, 0, 0, NULL};
  maskset seen = {w, 0, NULL};
  int64_t *stack = NULL, sp = 0, scap = 0;
  uint64_t *ext = calloc(w, sizeof(uint64_t));
  int rc = ORC_OK;
  if ((rc = mv_push(&vec, ext)) || (rc = ms_grow(&seen, &vec))) goto done;
  scap = 1024;
  stack = malloc(sizeof(int64_t) * scap);
  stack[sp++] = 0;
  while (sp) {
    int64_t li = stack[--sp];
    for (int v = 0; v < n; v++) {
      const uint64_t *lower = vec.masks + li * w; /* re-read: vec may move */
      int kw = v >> 6;
      uint64_t bit = 1ull << (v & 63);
      if (lower[kw] & bit) continue;
      const uint64_t *pv = g->preds + (size_t)v * w;
      int missing = 0;
      for (int q = 0; q < w && !missing; q++) missing = (pv[q] & ~lower[q]) != 0;
      if (missing) continue;
      memcpy(ext, lower, 8 * w);
      ext[kw] |= bit;
      uint64_t h = hash_mask(ext, w) & (seen.cap - 1);
      int found = 0;
      while (seen.slot[h] >= 0) {
        if (memcmp(vec.masks + seen.slot[h] * w, ext, 8 * w) == 0) { found = 1; break; }
        h = (h + 1) & (seen.cap - 1);
      }
      if (found) continue;
      if ((rc = mv_push(&vec, ext))) goto done;
      seen.slot[h] = vec.count - 1;
      if (vec.count > cap) { rc = ORC_ERR_LATTICE; goto done; }
      if (vec.count * 2 > seen.cap && (rc = ms_grow(&seen, &vec))) goto done;
      if (sp == scap) {
        scap *= 2;
        int64_t *ns = realloc(stack, sizeof(int64_t) * scap);
        if (!ns) { rc = ORC_ERR_NOMEM; goto done; }
        stack = ns;
      }
      stack[sp++] = vec.count - 1;
    }
  }
  sort_dedup(&vec);
done:
  free(ext);
  free(stack);
  free(seen.slot);
  if (rc) { free(vec.masks); return rc; }
  *out = vec;
  return ORC_OK;
}

/* pruned_lower_sets (lattice.py:87-93) with closures (graph.py:98-107) */
static int enumerate_pruned(const orc_graph *g, maskvec *out) {
  int n = g->n, w = g->w;
  maskvec vec = {w, 0, 0, NULL};
  uint64_t *clo = calloc((size_t)n * w, sizeof(uint64_t));
  uint64_t *tmp = calloc(w, sizeof(uint64_t));
  int rc = mv_push(&vec, tmp);
  full_set(n, w, tmp);
  if (!rc) rc = mv_push(&vec, tmp);
  for (int v = 0; v < n && !rc; v++) {
    uint64_t *c = clo + (size_t)v * w;
    c[v >> 6] |= 1ull << (v & 63);
    for (int k = 0; k < w; k++) {
      uint64_t x = g->preds[(size_t)v * w + k];
      while (x) {
        int u = k * 64 + __builtin_ctzll(x);
        x &= x - 1;
        for (int q = 0; q < w; q++) c[q] |= clo[(size_t)u * w + q];
      }
    }
    rc = mv_push(&vec, c);
  }
  free(clo);
  free(tmp);
  if (rc) { free(vec.masks); return rc; }
  sort_dedup(&vec);
  *out = vec;
  return ORC_OK;
}

static int build_family(const orc_graph *g, int family, int64_t cap, maskvec *out) {
  if (family == 1) return enumerate_pruned(g, out);
  if (family != 0) return ORC_ERR_ARG;
  return enumerate_full(g, cap, out);
}

int orc_family(const orc_graph *g, int family, int64_t cap, int64_t *size,
               uint64_t *masks_out, int64_t masks_cap) {
  maskvec fam;
  int rc = build_family(g, family, cap, &fam);
  if (rc) return rc;
  *size = fam.count;
  if (masks_out && fam.count <= masks_cap)
    memcpy(masks_out, fam.masks, sizeof(uint64_t) * g->w * fam.count);
  free(fam.masks);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* TransitionIndex (planner.py:95-136)                                       */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t j;
  int64_t stage_fixed, dt, dm;
} pair_t;

/* A cost vector restated as K weight classes: cost(S) = Σ_k value_k·|S ∩ C_k|
 * (an identity for any S when C_k = {v : cost_v = value_k}).  Used only when
 * the graph has ≤ 8 distinct costs; otherwise the bit loop of weight_of. */
typedef struct {
  int k;              /* 0 = not usable */
  int64_t value[8];
  uint64_t *mask;     /* [k][w] */
} wclass;

static void wclass_init(wclass *c, const int64_t *cost, int n, int w) {
  c->k = 0;
  c->mask = NULL;
  int k = 0;
  for (int v = 0; v < n; v++) {
    int f = 0;
    for (int q = 0; q < k; q++) f |= c->value[q] == cost[v];
    if (f) continue;
    if (k == 8) return;
    c->value[k++] = cost[v];
  }
  c->mask = calloc((size_t)(k ? k : 1) * w, sizeof(uint64_t));
  for (int v = 0; v < n; v++)
    for (int q = 0; q < k; q++)
      if (c->value[q] == cost[v]) c->mask[(size_t)q * w + (v >> 6)] |= 1ull << (v & 63);
  c->k = k;
}

static int64_t wclass_weight(const wclass *c, const int64_t *cost, const uint64_t *s, int w) {
  if (!c->k) return weight_of(cost, s, w);
  int64_t acc = 0;
  for (int q = 0; q < c->k; q++) {
    const uint64_t *m = c->mask + (size_t)q * w;
    int64_t cnt = 0;
    for (int k = 0; k < w; k++) cnt += __builtin_popcountll(s[k] & m[k]);
    acc += c->value[q] * cnt;
  }
  return acc;
}

typedef struct {
  const orc_graph *g;
  maskvec fam;
  uint64_t *bound;     /* [F][w] boundary(L_j)                    (109) */
  int64_t *stage_base; /* M(δ+(L)\L) + M(δ−(δ+(L))\L)           (110-115) */
  int64_t empty_index, full_index;
  pair_t **rows;       /* cached successor rows (NULL = not built) */
  wclass tcls, mcls;   /* T / M as weighted popcounts when few distinct costs */
  int32_t *row_len;
  int64_t cached_bytes, cache_limit;
} tindex;

static int index_materialise(tindex *ix);

static int index_init(tindex *ix, const orc_graph *g, maskvec fam) {
  int w = g->w;
  int64_t F = fam.count;
  ix->g = g;
  ix->fam = fam;
  ix->bound = malloc(sizeof(uint64_t) * w * F);
  ix->stage_base = malloc(sizeof(int64_t) * F);
  ix->rows = calloc(F, sizeof(pair_t *));
  ix->row_len = calloc(F, sizeof(int32_t));
  ix->cached_bytes = 0;
  ix->cache_limit = (int64_t)8 << 30;
  const char *lim = getenv("ORC_INDEX_CACHE_BYTES"); /* tests force the lazy path */
  if (lim) ix->cache_limit = atoll(lim);
  wclass_init(&ix->tcls, g->tcost, g->n, w);
  wclass_init(&ix->mcls, g->mcost, g->n, w);
  if (!ix->bound || !ix->stage_base || !ix->rows || !ix->row_len) return ORC_ERR_NOMEM;
#pragma omp parallel
  {
    uint64_t *succ = malloc(8 * w), *dm = malloc(8 * w), *tmp = malloc(8 * w);
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < F; i++) {
      const uint64_t *m = fam.masks + i * w;
      boundary(g, m, ix->bound + i * w);
      delta_plus(g, m, succ);
      for (int k = 0; k < w; k++) tmp[k] = succ[k] & ~m[k];
      int64_t a = weight_of(g->mcost, tmp, w);
      delta_minus(g, succ, dm);
      for (int k = 0; k < w; k++) tmp[k] = dm[k] & ~m[k];
      ix->stage_base[i] = a + weight_of(g->mcost, tmp, w);
    }
    free(succ); free(dm); free(tmp);
  }
  ix->empty_index = 0;           /* ∅ sorts first  */
  ix->full_index = F - 1;        /* V sorts last   */
  return index_materialise(ix);
}

static void index_free(tindex *ix) {
  if (ix->rows)
    for (int64_t i = 0; i < ix->fam.count; i++) free(ix->rows[i]);
  free(ix->rows);
  free(ix->row_len);
  free(ix->bound);
  free(ix->stage_base);
  free(ix->tcls.mask);
  free(ix->mcls.mask);
  free(ix->fam.masks);
}

/* Pair constants of L_i ⊆ L_j from their definitions (planner.py:124-131):
 * stage_fixed = 2·M(L_j\L_i) + stage_base[j], dt = T((L_j\L_i)\∂L_j),
 * dm = M(∂L_j\L_i). */
static void pair_constants(const tindex *ix, int64_t i, int64_t j, uint64_t *seg,
                           uint64_t *tmp, pair_t *p) {
  const orc_graph *g = ix->g;
  int w = g->w;
  const uint64_t *lo = ix->fam.masks + i * w, *hi = ix->fam.masks + j * w;
  const uint64_t *bj = ix->bound + j * w;
  for (int k = 0; k < w; k++) seg[k] = hi[k] & ~lo[k];
  p->j = (int32_t)j;
  p->stage_fixed = 2 * wclass_weight(&ix->mcls, g->mcost, seg, w) + ix->stage_base[j];
  for (int k = 0; k < w; k++) tmp[k] = seg[k] & ~bj[k];
  p->dt = wclass_weight(&ix->tcls, g->tcost, tmp, w);
  for (int k = 0; k < w; k++) tmp[k] = bj[k] & ~lo[k];
  p->dm = wclass_weight(&ix->mcls, g->mcost, tmp, w);
}

/* Successor row of member i: every j > i with L_i ⊆ L_j, with the reference's
 * pair constants (planner.py:118-131) evaluated from their definitions.
 * Serial; callers parallelise across rows.  Returns the row length; writes
 * the pairs when `row` is non-NULL. */
static int32_t build_row(const tindex *ix, int64_t i, pair_t *row) {
  const orc_graph *g = ix->g;
  int w = g->w;
  int64_t F = ix->fam.count;
  const uint64_t *lo = ix->fam.masks + i * w;
  uint64_t seg[64], tmp[64]; /* w <= 64 (n <= 4096) */
  int32_t cnt = 0;
  for (int64_t j = i + 1; j < F; j++) {
    const uint64_t *hi = ix->fam.masks + j * w;
    int sub = 1;
    for (int k = 0; k < w && sub; k++) sub = (lo[k] & ~hi[k]) == 0;
    if (!sub) continue;
    if (row) pair_constants(ix, i, j, seg, tmp, &row[cnt]);
    cnt++;
  }
  return cnt;
}

/* Materialise the whole index up front, as the reference does, when it fits
 * in `cache_limit` bytes (one parallel region across rows). */
static int index_materialise(tindex *ix) {
  int64_t F = ix->fam.count;
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : total)
  for (int64_t i = 0; i < F; i++) {
    ix->row_len[i] = build_row(ix, i, NULL);
    total += ix->row_len[i];
  }
  if (total * (int64_t)sizeof(pair_t) > ix->cache_limit) return ORC_OK; /* lazy rows */
  int fail = 0;
  for (int64_t i = 0; i < F; i++) {
    ix->rows[i] = malloc(sizeof(pair_t) * (ix->row_len[i] ? ix->row_len[i] : 1));
    if (!ix->rows[i]) fail = 1;
  }
  if (fail) return ORC_ERR_NOMEM;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < F; i++) build_row(ix, i, ix->rows[i]);
  ix->cached_bytes = total * (int64_t)sizeof(pair_t);
  return ORC_OK;
}


/* ------------------------------------------------------------------------ */
/* strategy.py: make_sequence + peak_memory                                  */
/* ------------------------------------------------------------------------ */

static int evaluate_chain(const orc_graph *g, int k, const uint64_t *chain,
                          int64_t *overhead, int64_t *stage_memory, int64_t *peak,
                          int64_t *cached_total) {
  int w = g->w, n = g->n;
  if (k < 1) return ORC_ERR_ARG;
  uint64_t *prev = calloc(w, 8), *acc = calloc(w, 8), *seg = malloc(8 * w),
           *bd = malloc(8 * w), *succ = malloc(8 * w), *dm = malloc(8 * w),
           *tmp = malloc(8 * w), *full = malloc(8 * w), *prev_cached = calloc(w, 8);
  full_set(n, w, full);
  int rc = ORC_OK;
  int64_t stagewise = 0, pk = 0;
  for (int i = 0; i < k && !rc; i++) {
    const uint64_t *m = chain + (size_t)i * w;
    /* make_sequence validation (strategy.py:74-83) */
    if (!is_lower_set(g, m)) { rc = ORC_ERR_ARG; break; }
    int inc = 1, eq = 1;
    for (int q = 0; q < w; q++) {
      inc &= (prev[q] & ~m[q]) == 0;
      eq &= prev[q] == m[q];
    }
    if (!inc || eq) { rc = ORC_ERR_ARG; break; }
    for (int q = 0; q < w; q++) seg[q] = m[q] & ~prev[q];
    boundary(g, m, bd);
    for (int q = 0; q < w; q++) acc[q] |= bd[q];
    /* overhead, stage-wise term (strategy.py:95-99) */
    for (int q = 0; q < w; q++) tmp[q] = seg[q] & ~bd[q];
    stagewise += weight_of(g->tcost, tmp, w);
    /* stage_memories (strategy.py:104-117) */
    delta_plus(g, m, succ);
    for (int q = 0; q < w; q++) tmp[q] = succ[q] & ~m[q];
    int64_t mem = weight_of(g->mcost, prev_cached, w) + 2 * weight_of(g->mcost, seg, w) +
                  weight_of(g->mcost, tmp, w);
    delta_minus(g, succ, dm);
    for (int q = 0; q < w; q++) tmp[q] = dm[q] & ~m[q];
    mem += weight_of(g->mcost, tmp, w);
    stage_memory[i] = mem;
    if (i == 0 || mem > pk) pk = mem;
    memcpy(prev_cached, acc, 8 * w);
    memcpy(prev, m, 8 * w);
  }
  if (!rc) {
    for (int q = 0; q < w; q++)
      if (prev[q] != full[q]) rc = ORC_ERR_ARG; /* must end at V (84-85) */
  }
  if (!rc) {
    for (int q = 0; q < w; q++) tmp[q] = full[q] & ~acc[q];
    int64_t total = weight_of(g->tcost, tmp, w);
    if (total != stagewise) rc = ORC_ERR_ASSERT; /* strategy.py:100 */
    *overhead = total;
    *peak = pk;
    *cached_total = weight_of(g->mcost, acc, w);
  }
  free(prev); free(acc); free(seg); free(bd); free(succ); free(dm); free(tmp);
  free(full); free(prev_cached);
  return rc;
}

int orc_evaluate(const orc_graph *g, int k, const uint64_t *chain,
                 int64_t *overhead, int64_t *stage_memory, int64_t *peak,
                 int64_t *cached_total) {
  return evaluate_chain(g, k, chain, overhead, stage_memory, peak, cached_total);
}

/* ------------------------------------------------------------------------ */
/* _dp_run / _reconstruct / _plan_with_index (planner.py:145-211)            */
/* ------------------------------------------------------------------------ */

static int plan_with_index(tindex *ix, int64_t budget, int objective, orc_plan *out) {
  const orc_graph *g = ix->g;
  int w = g->w;
  int64_t F = ix->fam.count;
  int64_t TV = 0;
  for (int v = 0; v < g->n; v++) TV += g->tcost[v];
  if (TV > (int64_t)1 << 28) return ORC_ERR_ARG; /* dense rows: keep T(V) sane */
  int64_t R = TV + 1;
  int minimize = objective == 0;
  orc_stats st = {0, 0, 0, 0};

  /* opt[i] (DpTable.opt) as dense rows, allocated when first touched */
  int64_t **opt = calloc(F, sizeof(int64_t *));
  int32_t **par_i = calloc(F, sizeof(int32_t *));
  int32_t **par_t = calloc(F, sizeof(int32_t *));
  int64_t *ft = malloc(sizeof(int64_t) * R), *fm = malloc(sizeof(int64_t) * R);
  if (!opt || !par_i || !par_t || !ft || !fm) return ORC_ERR_NOMEM;
  int rc = ORC_OK;
#define TOUCH(j)                                                             \
  do {                                                                       \
    if (!opt[j]) {                                                           \
      opt[j] = malloc(sizeof(int64_t) * R);                                  \
      par_i[j] = malloc(sizeof(int32_t) * R);                                \
      par_t[j] = malloc(sizeof(int32_t) * R);                                \
      for (int64_t q = 0; q < R; q++) opt[j][q] = EMPTY;                     \
    }                                                                        \
  } while (0)
  TOUCH(ix->empty_index);
  opt[ix->empty_index][0] = 0;
  par_i[ix->empty_index][0] = -1;
  int64_t pairs = 0;

  for (int64_t i = 0; i < F; i++) {
    int64_t *cell = opt[i];
    if (!cell) continue;
    /* frontier: strict prefix-min of m in t order (153-161) */
    int64_t nf = 0, best = EMPTY;
    int have = 0;
    for (int64_t q = 0; q < R; q++) {
      int64_t t = minimize ? q : R - 1 - q;
      int64_t m = cell[t];
      if (m == EMPTY) continue;
      if (have && m >= best) { st.dominated_skipped++; continue; }
      have = 1;
      best = m;
      ft[nf] = t;
      fm[nf] = m;
      nf++;
    }
    if (!have) continue;
    st.states_visited += nf;
    if (!ix->rows[i]) {
      /* lazy row (index too large to cache): the pair scan of build_row fused
       * with the relaxation, parallel over j (each target j has one writer) */
      int64_t cnt = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : cnt)
      for (int64_t j = i + 1; j < F; j++) {
        const uint64_t *lo = ix->fam.masks + i * w, *hi = ix->fam.masks + j * w;
        int sub = 1;
        for (int k = 0; k < w && sub; k++) sub = (lo[k] & ~hi[k]) == 0;
        if (!sub) continue;
        uint64_t seg[64], tmp[64];
        pair_t p;
        pair_constants(ix, i, j, seg, tmp, &p);
        cnt++;
        TOUCH(j);
        int64_t *target = opt[j];
        for (int64_t e = 0; e < nf; e++) {
          int64_t m = fm[e];
          if (m + p.stage_fixed > budget) continue;
          int64_t t2 = ft[e] + p.dt;
          int64_t m2 = m + p.dm;
          if (m2 < target[t2]) {
            target[t2] = m2;
            par_i[j][t2] = (int32_t)i;
            par_t[j][t2] = (int32_t)ft[e];
          }
        }
      }
      pairs += cnt;
      st.transitions += nf * cnt; /* counted before the budget test (164) */
      continue;
    }
    int32_t rl = ix->row_len[i];
    pair_t *row = ix->rows[i];
    pairs += rl;
    st.transitions += nf * (int64_t)rl; /* counted before the budget test (164) */
    for (int32_t r = 0; r < rl; r++) TOUCH(row[r].j);
    /* relax (165-175): targets are distinct per j, so j-parallel is exact */
#pragma omp parallel for schedule(dynamic, 64) if ((int64_t)rl * nf > (1 << 18))
    for (int32_t r = 0; r < rl; r++) {
      const pair_t p = row[r];
      int64_t *target = opt[p.j];
      for (int64_t e = 0; e < nf; e++) {
        int64_t m = fm[e];
        if (m + p.stage_fixed > budget) continue;
        int64_t t2 = ft[e] + p.dt;
        int64_t m2 = m + p.dm;
        if (m2 < target[t2]) {
          target[t2] = m2;
          par_i[p.j][t2] = (int32_t)i;
          par_t[p.j][t2] = (int32_t)ft[e];
        }
      }
    }
  }
  /* cells created by a passing transition are never empty (171-174) */
  for (int64_t i = 0; i < F; i++) {
    if (!opt[i]) continue;
    for (int64_t q = 0; q < R; q++) st.table_entries += opt[i][q] != EMPTY;
  }
  out->stats = st;
  out->family_size = F;
  out->pairs_expanded = pairs;
  out->feasible = 0;
  out->k = 0;

  int64_t *final = opt[ix->full_index];
  int64_t tstar = -1;
  if (!rc && final) {
    for (int64_t q = 0; q < R; q++) {
      int64_t t = minimize ? q : R - 1 - q;
      if (final[t] != EMPTY) { tstar = t; break; }
    }
  }
  if (!rc && tstar >= 0) {
    /* _reconstruct (180-189) */
    int64_t ci = ix->full_index, ct = tstar;
    int32_t len = 0;
    int64_t *path = calloc(g->n + 2, sizeof(int64_t));
    while (ci >= 0) {
      if (len > g->n + 1) { rc = ORC_ERR_ASSERT; break; }
      path[len++] = ci;
      int32_t pi = par_i[ci][ct];
      int32_t pt = par_t[ci][ct];
      ci = pi;
      ct = pt;
    }
    if (!rc && path[len - 1] != ix->empty_index) rc = ORC_ERR_ASSERT;
    if (!rc) {
      int k = len - 1;
      for (int s = 0; s < k; s++)
        memcpy(out->chain + (size_t)s * w, ix->fam.masks + path[len - 2 - s] * w, 8 * w);
      out->k = k;
      int64_t ovh, pk, ct2;
      rc = evaluate_chain(g, k, out->chain, &ovh, out->stage_memory, &pk, &ct2);
      if (!rc) {
        /* self-checks (206-210) */
        if (ovh != tstar || pk > budget || ct2 != final[tstar]) rc = ORC_ERR_ASSERT;
        out->feasible = 1;
        out->t_star = tstar;
        out->overhead = ovh;
        out->peak = pk;
        out->cached_total = ct2;
      }
    }
    free(path);
  }
  for (int64_t i = 0; i < F; i++) { free(opt[i]); free(par_i[i]); free(par_t[i]); }
  free(opt); free(par_i); free(par_t); free(ft); free(fm);
  if (rc) return rc;
  return out->feasible ? ORC_OK : ORC_INFEASIBLE;
#undef TOUCH
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int orc_dp_plan(const orc_graph *g, int family, int64_t cap, int64_t budget,
                int objective, int nthreads, orc_plan *out) {
  if (budget < 0 || (objective != 0 && objective != 1)) return ORC_ERR_ARG;
  set_threads(nthreads);
  maskvec fam;
  int rc = build_family(g, family, cap, &fam);
  if (rc) return rc;
  tindex ix;
  memset(&ix, 0, sizeof ix);
  double t0 = now_s();
  rc = index_init(&ix, g, fam);
  double t1 = now_s();
  if (!rc) rc = plan_with_index(&ix, budget, objective, out);
  if (getenv("ORC_VERBOSE"))
    fprintf(stderr, "orc_dp_plan: F=%lld index %.3f s, dp %.3f s\n", (long long)fam.count,
            t1 - t0, now_s() - t1);
  index_free(&ix);
  return rc;
}

int orc_min_feasible_budget(const orc_graph *g, int family, int64_t cap,
                            int objective, int nthreads, int64_t *b_min,
                            orc_plan *out, int64_t *probes,
                            int64_t *probe_transitions) {
  set_threads(nthreads);
  maskvec fam;
  int rc = build_family(g, family, cap, &fam);
  if (rc) return rc;
  tindex ix;
  memset(&ix, 0, sizeof ix);
  rc = index_init(&ix, g, fam);
  int64_t MV = 0;
  for (int v = 0; v < g->n; v++) MV += g->mcost[v];
  int64_t hi = 2 * MV, lo = 0;
  *probes = 0;
  *probe_transitions = 0;
  /* scratch plan buffers for probes that do not end up as the answer */
  uint64_t *chain2 = malloc(sizeof(uint64_t) * g->w * (g->n + 1));
  int64_t *stage2 = malloc(sizeof(int64_t) * (g->n + 1));
  orc_plan probe = *out;
  probe.chain = chain2;
  probe.stage_memory = stage2;
  if (!rc) {
    rc = plan_with_index(&ix, hi, objective, out);
    (*probes)++;
    *probe_transitions += out->stats.transitions;
    if (rc == ORC_INFEASIBLE) rc = ORC_ERR_PLANNER; /* planner.py:287-288 */
  }
  while (!rc && hi - lo > 1) {
    int64_t mid = (lo + hi) / 2;
    int prc = plan_with_index(&ix, mid, objective, &probe);
    (*probes)++;
    *probe_transitions += probe.stats.transitions;
    if (prc == ORC_OK) {
      hi = mid;
      uint64_t *c = out->chain;
      int64_t *s = out->stage_memory;
      memcpy(c, probe.chain, sizeof(uint64_t) * g->w * probe.k);
      memcpy(s, probe.stage_memory, sizeof(int64_t) * probe.k);
      *out = probe;
      out->chain = c;
      out->stage_memory = s;
    } else if (prc == ORC_INFEASIBLE) {
      lo = mid;
    } else {
      rc = prc;
    }
  }
  *b_min = hi;
  free(chain2);
  free(stage2);
  index_free(&ix);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* simulate (schedule.py:184-254)                                            */
/* ------------------------------------------------------------------------ */

int orc_simulate(const orc_graph *g, int64_t nops, const int32_t *ops,
                 int64_t *trace, orc_sim_result *out) {
  int n = g->n, w = g->w;
  uint64_t *fwd = calloc(w, 8), *grad = calloc(w, 8);
  int32_t *runs = calloc(n > 0 ? n : 1, sizeof(int32_t));
  int64_t mem = 0, peak = 0, total = 0, rec = 0, back = 0;
  int rc = ORC_OK;
  out->err_idx = -1;
  out->err_code = 0;
  out->err_v = out->err_w = -1;
#define FAIL(code, v_, w_)             \
  do {                                 \
    out->err_idx = idx;                \
    out->err_code = (code);            \
    out->err_v = (v_);                 \
    out->err_w = (w_);                 \
    rc = ORC_ERR_SIM;                  \
    goto done;                         \
  } while (0)
  for (int64_t idx = 0; idx < nops; idx++) {
    int kind = ops[2 * idx], v = ops[2 * idx + 1];
    if (v < 0 || v >= n || kind < 0 || kind > 3) { rc = ORC_ERR_ARG; goto done; }
    uint64_t bit = 1ull << (v & 63);
    int kw = v >> 6;
    if (kind == 0) {
      const uint64_t *pv = g->preds + (size_t)v * w;
      for (int q = 0; q < w; q++) {
        uint64_t miss = pv[q] & ~fwd[q];
        if (miss) FAIL(1, v, q * 64 + __builtin_ctzll(miss));
      }
      if (fwd[kw] & bit) FAIL(2, v, -1);
      runs[v]++;
      if (runs[v] > 2) FAIL(3, v, -1);
      if (runs[v] == 2) rec += g->tcost[v];
      total += g->tcost[v];
      fwd[kw] |= bit;
      mem += g->mcost[v];
    } else if (kind == 1) {
      const uint64_t *pv = g->preds + (size_t)v * w;
      for (int q = 0; q < w; q++) {
        uint64_t need = pv[q] | (q == kw ? bit : 0);
        uint64_t miss = need & ~fwd[q];
        if (miss) FAIL(4, v, q * 64 + __builtin_ctzll(miss));
      }
      const uint64_t *sv = g->succs + (size_t)v * w;
      for (int q = 0; q < w; q++) {
        uint64_t miss = sv[q] & ~grad[q];
        if (miss) FAIL(5, v, q * 64 + __builtin_ctzll(miss));
      }
      if (grad[kw] & bit) FAIL(6, v, -1);
      grad[kw] |= bit;
      mem += g->mcost[v];
      back++;
    } else if (kind == 2) {
      if (!(fwd[kw] & bit)) FAIL(7, v, -1);
      fwd[kw] ^= bit;
      mem -= g->mcost[v];
    } else {
      if (!(grad[kw] & bit)) FAIL(8, v, -1);
      grad[kw] ^= bit;
      mem -= g->mcost[v];
    }
    if (mem > peak) peak = mem;
    if (trace) trace[idx] = mem;
  }
done:
#undef FAIL
  out->peak = peak;
  out->total_forward = total;
  out->recompute = rec;
  out->backward_count = back;
  free(fwd); free(grad); free(runs);
  return rc;
}
