/* TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * Plain-C restatement of the reference hot path. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Deliberately naive (sequential, sort-based, per-edge log1p) so that it reads
 * like the reference and not like the CUDA library it checks.
 */
#define _GNU_SOURCE
#include "vipkit_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* vp_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ rng */
/* mix64: splitmix64 finalizer, include/vipkit/rng.hpp:9-14 */
uint64_t vp_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
/* RngStream ctor, rng.hpp:21 */
void vp_stream_init(vp_stream* s, uint64_t key) { s->counter = vp_mix64(key); }
/* RngStream::next_u64, rng.hpp:23-29 (Weyl counter then the finalizer) */
uint64_t vp_next_u64(vp_stream* s) {
  s->counter += 0x9e3779b97f4a7c15ull;
  uint64_t x = s->counter;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
/* rng.hpp:32 */
double vp_next_double(vp_stream* s) { return (double)(vp_next_u64(s) >> 11) * 0x1.0p-53; }
/* rng.hpp:35-40: rejection below limit = ~0 - ~0 % bound, then modulo */
uint64_t vp_next_below(vp_stream* s, uint64_t bound) {
  const uint64_t limit = ~0ull - ~0ull % bound;
  uint64_t x = vp_next_u64(s);
  while (x >= limit) x = vp_next_u64(s);
  return x % bound;
}
/* SeedSpec::key, rng.hpp:63-67 */
uint64_t vp_seed_key(uint64_t seed, const uint64_t* parts, uint32_t np) {
  uint64_t h = seed;
  for (uint32_t i = 0; i < np; ++i) h = vp_mix64(h ^ vp_mix64(parts[i]));
  return h;
}
/* SeedSpec::derived, rng.hpp:61 */
uint64_t vp_seed_derived(uint64_t seed, uint64_t tag) { return vp_mix64(seed ^ vp_mix64(tag)); }

void vp_free(void* p) { free(p); }

/* `count` draws of one stream: next_below(bound), or next_u64 when bound == 0 */
void vp_stream_draws(uint64_t key, uint64_t bound, uint64_t count, uint64_t* out) {
  vp_stream s;
  vp_stream_init(&s, key);
  for (uint64_t i = 0; i < count; ++i) out[i] = bound ? vp_next_below(&s, bound) : vp_next_u64(&s);
}

/* ---------------------------------------------------------------- graph */
typedef struct { uint32_t u, v; } edge_t;
static int cmp_edge(const void* a, const void* b) {
  const edge_t* x = a;
  const edge_t* y = b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}

/* Graph::from_edges forward side, graph.cpp:33-48 (symmetrize, drop
 * self-loops, sort, unique) + build_csr graph.cpp:18-29. */
int vp_graph_from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst, uint64_t ne,
                        int undirected, uint64_t** off_out, uint32_t** tgt_out, uint64_t* m_out) {
  if (n == 0 || n > (1ull << 32)) return fail(2, "vertex count out of range");
  uint64_t cap = undirected ? 2 * ne : ne;
  edge_t* e = malloc((cap ? cap : 1) * sizeof(edge_t));
  uint64_t k = 0;
  for (uint64_t i = 0; i < ne; ++i)
    if (src[i] != dst[i]) e[k++] = (edge_t){src[i], dst[i]};
  if (undirected)
    for (uint64_t i = 0; i < ne; ++i)
      if (src[i] != dst[i]) e[k++] = (edge_t){dst[i], src[i]};
  qsort(e, k, sizeof(edge_t), cmp_edge);
  uint64_t m = 0;
  for (uint64_t i = 0; i < k; ++i)
    if (m == 0 || cmp_edge(&e[m - 1], &e[i]) != 0) e[m++] = e[i];
  uint64_t* off = calloc(n + 1, 8);
  uint32_t* tgt = malloc((m ? m : 1) * 4);
  for (uint64_t i = 0; i < m; ++i) off[e[i].u + 1]++;
  for (uint64_t i = 0; i < n; ++i) off[i + 1] += off[i];
  for (uint64_t i = 0; i < m; ++i) tgt[i] = e[i].v; /* already sorted per source */
  free(e);
  *off_out = off;
  *tgt_out = tgt;
  *m_out = m;
  return VP_OK;
}

typedef struct {
  uint32_t* u;
  uint32_t* v;
  uint64_t n, cap;
} elist;
static void el_push(elist* l, uint32_t u, uint32_t v) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 1024;
    l->u = realloc(l->u, l->cap * 4);
    l->v = realloc(l->v, l->cap * 4);
  }
  l->u[l->n] = u;
  l->v[l->n] = v;
  l->n++;
}

/* generate_synthetic, graph.cpp:139-245 */
int vp_generate(int kind, uint64_t n, uint64_t d, uint64_t seed, uint64_t** off, uint32_t** tgt,
                uint64_t* m) {
  if (n < 1) return fail(VP_PARAMETER, "synthetic graph needs n >= 1");
  elist el = {0};
  switch (kind) {
    case VP_PATH: /* graph.cpp:139-144 */
      for (uint64_t i = 0; i + 1 < n; ++i) el_push(&el, (uint32_t)i, (uint32_t)(i + 1));
      break;
    case VP_STAR: /* graph.cpp:146-150 */
      for (uint64_t i = 1; i < n; ++i) el_push(&el, 0, (uint32_t)i);
      break;
    case VP_TREE: /* graph.cpp:152-157 */
      if (d < 1) return fail(VP_PARAMETER, "tree arity must be >= 1");
      for (uint64_t i = 1; i < n; ++i) el_push(&el, (uint32_t)((i - 1) / d), (uint32_t)i);
      break;
    case VP_GRID: /* graph.cpp:159-167 */
      if (d < 1) return fail(VP_PARAMETER, "grid column count must be >= 1");
      for (uint64_t i = 0; i < n; ++i) {
        if ((i + 1) % d != 0 && i + 1 < n) el_push(&el, (uint32_t)i, (uint32_t)(i + 1));
        if (i + d < n) el_push(&el, (uint32_t)i, (uint32_t)(i + d));
      }
      break;
    case VP_PA: { /* graph.cpp:173-203 */
      if (d < 1) return fail(VP_PARAMETER, "attachment degree must be >= 1");
      uint64_t parts[2] = {0xA1, 1};
      vp_stream rng;
      vp_stream_init(&rng, vp_seed_key(seed, parts, 2));
      uint32_t* endpoints = malloc(2 * n * d * 4 + 4);
      uint64_t ne = 0;
      uint32_t* chosen = malloc(d * 4);
      for (uint64_t v = 1; v < n; ++v) {
        const uint64_t dv = d < v ? d : v;
        uint64_t nc = 0;
        for (uint64_t j = 0; j < dv; ++j) {
          uint32_t t;
          int again;
          do {
            t = ne == 0 ? (uint32_t)vp_next_below(&rng, v) : endpoints[vp_next_below(&rng, ne)];
            again = (t == v);
            for (uint64_t c = 0; c < nc && !again; ++c) again = (chosen[c] == t);
          } while (again);
          chosen[nc++] = t;
        }
        for (uint64_t c = 0; c < nc; ++c) {
          el_push(&el, (uint32_t)v, chosen[c]);
          endpoints[ne++] = (uint32_t)v;
          endpoints[ne++] = chosen[c];
        }
      }
      free(chosen);
      free(endpoints);
      uint32_t* relabel = malloc(n * 4);
      for (uint64_t v = 0; v < n; ++v) relabel[v] = (uint32_t)v;
      for (uint64_t i = n; i > 1; --i) {
        const uint64_t j = vp_next_below(&rng, i);
        const uint32_t t = relabel[i - 1];
        relabel[i - 1] = relabel[j];
        relabel[j] = t;
      }
      for (uint64_t i = 0; i < el.n; ++i) {
        el.u[i] = relabel[el.u[i]];
        el.v[i] = relabel[el.v[i]];
      }
      free(relabel);
      break;
    }
    case VP_UNIFORM: { /* graph.cpp:205-216 */
      if (d < 1) return fail(VP_PARAMETER, "edges-per-vertex must be >= 1");
      uint64_t parts[2] = {0xA1, 2};
      vp_stream rng;
      vp_stream_init(&rng, vp_seed_key(seed, parts, 2));
      for (uint64_t i = 0; i < n * d; ++i) {
        const uint32_t u = (uint32_t)vp_next_below(&rng, n);
        const uint32_t v = (uint32_t)vp_next_below(&rng, n);
        if (u != v) el_push(&el, u, v);
      }
      break;
    }
    default:
      return fail(VP_PARAMETER, "unknown synthetic graph kind");
  }
  const int rc = vp_graph_from_edges(n, el.u, el.v, el.n, 1, off, tgt, m);
  free(el.u);
  free(el.v);
  return rc;
}

/* make_roles, graph.cpp:247-268 */
int vp_make_roles(uint64_t n, double train, double valid, double test, uint64_t seed, uint8_t* out) {
  if (train < 0 || valid < 0 || test < 0 || train + valid + test > 1.0 + 1e-12)
    return fail(VP_PARAMETER, "role fractions must be non-negative and sum to <= 1");
  uint32_t* order = malloc((n ? n : 1) * 4);
  for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  uint64_t parts[1] = {0xA2};
  vp_stream rng;
  vp_stream_init(&rng, vp_seed_key(seed, parts, 1));
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = vp_next_below(&rng, i);
    const uint32_t t = order[i - 1];
    order[i - 1] = order[j];
    order[j] = t;
  }
  memset(out, 3, n);
  const uint64_t t = (uint64_t)(train * (double)n);
  const uint64_t va = (uint64_t)(valid * (double)n);
  const uint64_t te = (uint64_t)(test * (double)n);
  uint64_t i = 0;
  for (uint64_t j = 0; j < t && i < n; ++j, ++i) out[order[i]] = 0;
  for (uint64_t j = 0; j < va && i < n; ++j, ++i) out[order[i]] = 1;
  for (uint64_t j = 0; j < te && i < n; ++j, ++i) out[order[i]] = 2;
  free(order);
  return VP_OK;
}

/* ------------------------------------------------------------- sampling */
/* epoch_minibatches, sampling.cpp:45-70; train_members graph.cpp:106-111 */
int vp_epoch_minibatches(const uint8_t* roles, uint64_t n, const uint32_t* labels, uint32_t k,
                         uint64_t b, uint64_t epoch, uint64_t seed, uint32_t* out_perm,
                         uint64_t* out_count) {
  if (b == 0) return fail(VP_PARAMETER, "batch size must be >= 1");
  uint64_t T = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (labels[v] == k && roles[v] == 0) out_perm[T++] = (uint32_t)v;
  if (T == 0) return fail(VP_SAMPLING, "partition has no train vertices");
  uint64_t parts[3] = {0xB1, epoch, k};
  vp_stream rng;
  vp_stream_init(&rng, vp_seed_key(seed, parts, 3));
  for (uint64_t i = T; i > 1; --i) {
    const uint64_t j = vp_next_below(&rng, i);
    const uint32_t t = out_perm[i - 1];
    out_perm[i - 1] = out_perm[j];
    out_perm[j] = t;
  }
  *out_count = T;
  return VP_OK;
}

/* sample_neighbors, sampling.cpp:72-92 (full scratch copy + partial FY) */
uint64_t vp_sample_neighbors(const uint64_t* off, const uint32_t* tgt, uint32_t v, uint32_t fanout,
                             vp_stream* s, uint32_t* out) {
  const uint64_t deg = off[v + 1] - off[v];
  const uint32_t* nbrs = tgt + off[v];
  if (deg <= fanout) {
    memcpy(out, nbrs, deg * 4);
    return deg;
  }
  uint32_t* scratch = malloc(deg * 4);
  memcpy(scratch, nbrs, deg * 4);
  for (uint32_t i = 0; i < fanout; ++i) {
    const uint64_t j = i + vp_next_below(s, deg - i);
    const uint32_t t = scratch[i];
    scratch[i] = scratch[j];
    scratch[j] = t;
    out[i] = scratch[i];
  }
  free(scratch);
  return fanout;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}
static uint64_t sort_unique(uint32_t* a, uint64_t k) {
  qsort(a, k, 4, cmp_u32);
  uint64_t m = 0;
  for (uint64_t i = 0; i < k; ++i)
    if (m == 0 || a[m - 1] != a[i]) a[m++] = a[i];
  return m;
}

/* expand, sampling.cpp:94-128, plus the MFG edge list: per hop, sources in
 * the order expand visits them (hop 1 = batch order, later = sorted frontier)
 * and each source's draws in emission order (builder contract). */
vp_expansion* vp_expand(const uint64_t* off, const uint32_t* tgt, uint64_t n, const uint32_t* batch,
                        uint64_t nb, const uint32_t* fanouts, uint32_t L, uint64_t seed,
                        uint64_t epoch, uint32_t part, uint64_t batch_index) {
  (void)n;
  if (nb == 0) {
    fail(VP_SAMPLING, "cannot expand an empty batch");
    return NULL;
  }
  if (L == 0) {
    fail(VP_PARAMETER, "fanout list must have at least one hop");
    return NULL;
  }
  for (uint32_t h = 0; h < L; ++h)
    if (fanouts[h] < 1) {
      fail(VP_PARAMETER, "each fanout must be >= 1");
      return NULL;
    }
  vp_expansion* x = calloc(1, sizeof *x);
  x->L = L;
  x->nb = nb;
  x->batch = malloc(nb * 4);
  memcpy(x->batch, batch, nb * 4);
  x->fsize = calloc(L, 8);
  x->frontier = calloc(L, sizeof(uint32_t*));
  x->indptr = calloc(L, sizeof(uint64_t*));
  x->edges = calloc(L, sizeof(uint32_t*));
  const uint32_t* cur = x->batch;
  uint64_t ncur = nb;
  for (uint32_t h = 1; h <= L; ++h) {
    uint64_t cap = 0;
    for (uint64_t i = 0; i < ncur; ++i) {
      const uint64_t deg = off[cur[i] + 1] - off[cur[i]];
      cap += deg < fanouts[h - 1] ? deg : fanouts[h - 1];
    }
    uint32_t* ed = malloc((cap ? cap : 1) * 4);
    uint64_t* ip = malloc((ncur + 1) * 8);
    ip[0] = 0;
    uint64_t pos = 0;
    for (uint64_t i = 0; i < ncur; ++i) {
      uint64_t parts[6] = {0xB2, epoch, part, batch_index, h, cur[i]};
      vp_stream s;
      vp_stream_init(&s, vp_seed_key(seed, parts, 6));
      pos += vp_sample_neighbors(off, tgt, cur[i], fanouts[h - 1], &s, ed + pos);
      ip[i + 1] = pos;
    }
    x->indptr[h - 1] = ip;
    x->edges[h - 1] = ed;
    uint32_t* fr = malloc((pos ? pos : 1) * 4);
    memcpy(fr, ed, pos * 4);
    x->fsize[h - 1] = sort_unique(fr, pos);
    x->frontier[h - 1] = fr;
    cur = fr;
    ncur = x->fsize[h - 1];
  }
  uint64_t tot = nb;
  for (uint32_t h = 0; h < L; ++h) tot += x->fsize[h];
  x->all = malloc(tot * 4);
  memcpy(x->all, batch, nb * 4);
  uint64_t p = nb;
  for (uint32_t h = 0; h < L; ++h) {
    memcpy(x->all + p, x->frontier[h], x->fsize[h] * 4);
    p += x->fsize[h];
  }
  x->nall = sort_unique(x->all, tot);
  return x;
}

void vp_expansion_free(vp_expansion* x) {
  if (!x) return;
  for (uint32_t h = 0; h < x->L; ++h) {
    free(x->frontier[h]);
    free(x->indptr[h]);
    free(x->edges[h]);
  }
  free(x->frontier);
  free(x->indptr);
  free(x->edges);
  free(x->fsize);
  free(x->batch);
  free(x->all);
  free(x);
}

/* ------------------------------------------------------------------ vip */
/* initial_probs, vip.cpp:25-35 */
int vp_initial_probs(const uint8_t* roles, uint64_t n, const uint32_t* labels, uint32_t k,
                     uint64_t b, double* out) {
  if (b == 0) return fail(VP_PARAMETER, "batch size must be >= 1");
  uint64_t T = 0;
  for (uint64_t v = 0; v < n; ++v) T += (labels[v] == k && roles[v] == 0);
  if (T == 0) return fail(VP_SAMPLING, "partition has no train vertices");
  double p = (double)b / (double)T;
  if (p > 1.0) p = 1.0;
  for (uint64_t v = 0; v < n; ++v) out[v] = (labels[v] == k && roles[v] == 0) ? p : 0.0;
  return VP_OK;
}

/* clamp_prob, vip.cpp:16-21 */
static double clamp_prob(double x) {
  if (!(x > 1e-300)) return 0.0;
  return x < 1.0 ? x : 1.0;
}

/* propagate, vip.cpp:37-83 (hoist :57-61, per-edge log1p pull :62-72,
 * total :76-81); TransitionModel::weight vip.hpp:22-26 */
int vp_propagate(const uint64_t* fwd_off, const uint64_t* rev_off, const uint32_t* rev_tgt,
                 uint64_t n, const uint32_t* fanouts, uint32_t L, const double* p0,
                 double* hop_out, double* total_out) {
  if (L == 0) return fail(VP_PARAMETER, "fanout list must have at least one hop");
  for (uint32_t h = 0; h < L; ++h)
    if (fanouts[h] < 1) return fail(VP_PARAMETER, "each fanout must be >= 1");
  for (uint64_t v = 0; v < n; ++v)
    if (!(p0[v] >= 0.0 && p0[v] <= 1.0)) return fail(VP_PARAMETER, "p0 entries must lie in [0,1]");
  double* hop = hop_out ? hop_out : malloc(L * n * 8);
  double* sp = malloc((n ? n : 1) * 8);
  const double* prev = p0;
  for (uint32_t h = 1; h <= L; ++h) {
    double* cur = hop + (uint64_t)(h - 1) * n;
    const double f = (double)fanouts[h - 1];
    for (uint64_t v = 0; v < n; ++v) {
      const double pv = prev[v];
      const double d = (double)(fwd_off[v + 1] - fwd_off[v]);
      const double w = d <= f ? 1.0 : f / d;
      sp[v] = pv == 0.0 ? 0.0 : w * pv;
    }
    for (uint64_t u = 0; u < n; ++u) {
      double log_miss = 0.0;
      for (uint64_t i = rev_off[u]; i < rev_off[u + 1]; ++i) {
        const double wp = sp[rev_tgt[i]];
        if (wp == 0.0) continue;
        log_miss += log1p(-wp);
      }
      cur[u] = clamp_prob(-expm1(log_miss));
    }
    prev = cur;
  }
  for (uint64_t u = 0; u < n; ++u) {
    double log_miss = 0.0;
    for (uint32_t h = 0; h < L; ++h) log_miss += log1p(-hop[(uint64_t)h * n + u]);
    total_out[u] = clamp_prob(-expm1(log_miss));
  }
  free(sp);
  if (!hop_out) free(hop);
  return VP_OK;
}

/* ------------------------------------------------------------- policies */
static _Thread_local const double* g_scores;
/* order_remotes comparator, policies.cpp:26-30 (score desc, id asc) */
static int cmp_rank(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (g_scores[x] != g_scores[y]) return g_scores[x] > g_scores[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}

/* rank_by_scores -> order_remotes, policies.cpp:134-138, 20-34 */
int vp_rank_by_scores(const uint32_t* labels, uint64_t n, uint32_t k, const double* scores,
                      uint32_t* order_out, double* score_out, uint64_t* count) {
  uint64_t c = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (labels[v] != k) order_out[c++] = (uint32_t)v;
  g_scores = scores;
  qsort(order_out, c, 4, cmp_rank);
  for (uint64_t i = 0; i < c; ++i) score_out[i] = scores[order_out[i]];
  *count = c;
  return VP_OK;
}

/* build_cache capacity, policies.cpp:150-156 */
int vp_cache_capacity(double alpha, uint64_t n, uint32_t K, uint64_t* cap) {
  if (alpha < 0) return fail(VP_PARAMETER, "replication factor must be >= 0");
  if (K == 0) return fail(VP_PARAMETER, "need at least one ranking");
  *cap = (uint64_t)floor(alpha * (double)n / (double)K + 1e-9);
  return VP_OK;
}

/* classify, commsim.cpp:61-73; is_cached policies.hpp:58-60 */
void vp_classify(const uint32_t* all, uint64_t nall, const uint32_t* labels, uint32_t k,
                 const uint64_t* bits, uint64_t counts[3]) {
  counts[0] = counts[1] = counts[2] = 0;
  for (uint64_t i = 0; i < nall; ++i) {
    const uint32_t v = all[i];
    if (labels[v] == k)
      counts[0]++;
    else if (bits && ((bits[v >> 6] >> (v & 63)) & 1u))
      counts[1]++;
    else
      counts[2]++;
  }
}

/* build_reorder, reorder.cpp:11-34 */
int vp_build_reorder(const uint32_t* labels, uint64_t n, uint32_t K, const double* scores,
                     uint32_t* old_of_new, uint64_t* ranges) {
  uint64_t pos = 0;
  for (uint32_t k = 0; k < K; ++k) {
    const uint64_t start = pos;
    for (uint64_t v = 0; v < n; ++v)
      if (labels[v] == k) old_of_new[pos++] = (uint32_t)v;
    g_scores = scores + (uint64_t)k * n;
    qsort(old_of_new + start, pos - start, 4, cmp_rank);
    ranges[2 * k] = start;
    ranges[2 * k + 1] = pos;
  }
  return pos == n ? VP_OK : fail(VP_SHAPE, "labels out of range");
}

/* ------------------------------------------------------ synthetic features */
/* Builder contract: X[v][j] = top bits of mix64(seed ^
 * mix64(v*D + j)) mapped onto an exactly representable grid in [-1, 1):
 * 24 bits for fp32, 11 bits for fp16, so host and device agree bit-for-bit. */
static uint64_t feat_bits(uint64_t seed, uint64_t v, uint32_t j, uint32_t D) {
  return vp_mix64(seed ^ vp_mix64(v * (uint64_t)D + j));
}
float vp_feature_f32(uint64_t seed, uint64_t v, uint32_t j, uint32_t D) {
  return (float)(feat_bits(seed, v, j, D) >> 40) * 0x1.0p-23f - 1.0f;
}
uint16_t vp_feature_f16_bits(uint64_t seed, uint64_t v, uint32_t j, uint32_t D) {
  const float x = (float)(feat_bits(seed, v, j, D) >> 53) * 0x1.0p-10f - 1.0f; /* exact in fp16 */
  uint32_t b;
  memcpy(&b, &x, 4);
  const uint32_t sign = (b >> 16) & 0x8000u;
  const uint32_t absb = b & 0x7fffffffu;
  if (absb == 0) return (uint16_t)sign;
  const int exp = (int)(absb >> 23) - 127;       /* |x| >= 2^-10 here: normal in fp16 */
  const uint32_t mant = (absb & 0x7fffffu) >> 13; /* low 13 bits are zero by construction */
  return (uint16_t)(sign | (uint32_t)(exp + 15) << 10 | mant);
}
void vp_features(uint64_t seed, uint32_t D, int fp16, const uint32_t* ids, uint64_t count,
                 void* out) {
  for (uint64_t i = 0; i < count; ++i)
    for (uint32_t j = 0; j < D; ++j) {
      if (fp16)
        ((uint16_t*)out)[i * D + j] = vp_feature_f16_bits(seed, ids[i], j, D);
      else
        ((float*)out)[i * D + j] = vp_feature_f32(seed, ids[i], j, D);
    }
}
