/* TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * Host-side workload pieces for the CPU arms of bench.py and for tests, so
 * that neither the reference arm (`bench.py --impl reference`) nor the CPU
 * baseline needs the product library:
 *
 *  - vp_synth_community_powerlaw: plain-C restatement of the bench's graph
 *    recipe (the builder-defined community power-law generator, DESIGN.md §6;
 *    product: vk_synth_community_powerlaw in csrc/capi.cu). The output is the
 *    canonical CSR of Graph::from_edges (graph.cpp:33-53: symmetrised,
 *    self-loops dropped, rows sorted and deduplicated), so it is identical for
 *    any thread count; tests/test_bench_arms.py pins it to the product's.
 *  - vp_fill_features / vp_gather_rows: the counter-hashed feature table
 *     and the CPU row gather out[i] = X[ids[i]] the GPU gather is
 *    measured against (the reference never materialises features,
 *    SPEC.md:157, so this is a labelled restatement, not reference code).
 *
 * pthreads, one contiguous row range per worker.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>

#include "vipkit_port.h"

/* key fold step of SeedSpec::key, rng.hpp:63-67 */
static uint64_t key_step(uint64_t h, uint64_t part) { return vp_mix64(h ^ vp_mix64(part)); }

typedef void (*range_fn)(void* ctx, uint64_t lo, uint64_t hi);
typedef struct {
  range_fn fn;
  void* ctx;
  uint64_t lo, hi;
} range_job;
static void* range_main(void* a) {
  range_job* j = a;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}
static void parallel_rows(unsigned T, uint64_t n, range_fn fn, void* ctx) {
  if (T < 1) T = 1;
  pthread_t* th = malloc(sizeof(pthread_t) * T);
  range_job* jb = malloc(sizeof(range_job) * T);
  for (unsigned t = 0; t < T; ++t) {
    jb[t] = (range_job){fn, ctx, n * t / T, n * (t + 1) / T};
    pthread_create(&th[t], NULL, range_main, &jb[t]);
  }
  for (unsigned t = 0; t < T; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jb);
}

/* ------------------------------------------------- community power-law graph */
typedef struct {
  uint64_t n, d, base_key;
  uint32_t C;
  double p_in, skew;
  uint32_t *rank_to_vertex, *vertex_to_rank;
  uint32_t* deg;     /* pass 1 (atomic) */
  uint64_t* off;     /* raw multigraph offsets */
  uint64_t* cur;     /* pass 2 cursors (atomic) */
  uint32_t* slots;
  uint64_t* newdeg;
  uint64_t* o;       /* final offsets */
  uint32_t* t;       /* final targets */
} gen_ctx;

static uint64_t cstart(const gen_ctx* g, uint32_t c) { return (uint64_t)c * g->n / g->C; }
static uint32_t comm_of_rank(const gen_ctx* g, uint64_t r) {
  uint32_t c = (uint32_t)((r * g->C) / g->n);
  while (c + 1 < g->C && cstart(g, c + 1) <= r) ++c;
  while (cstart(g, c) > r) --c;
  return c;
}
/* stub (u, j): own stream key (0xA1, 3, u, j); target community = own with
 * probability p_in else uniform; target = member of popularity rank
 * floor(size * U^skew) */
static uint32_t stub(const gen_ctx* g, uint64_t u, uint64_t j) {
  vp_stream s;
  vp_stream_init(&s, key_step(key_step(g->base_key, u), j));
  const uint32_t cu = comm_of_rank(g, g->vertex_to_rank[u]);
  const double a = vp_next_double(&s);
  const uint32_t c = a < g->p_in ? cu : (uint32_t)vp_next_below(&s, g->C);
  const uint64_t lo = cstart(g, c), size = cstart(g, c + 1) - lo;
  const double x = vp_next_double(&s);
  uint64_t r = (uint64_t)((double)size * (g->skew == 2.0 ? x * x : pow(x, g->skew)));
  if (r >= size) r = size - 1;
  return g->rank_to_vertex[lo + r];
}
static void pass_degrees(void* p, uint64_t lo, uint64_t hi) {
  gen_ctx* g = p;
  for (uint64_t u = lo; u < hi; ++u)
    for (uint64_t j = 0; j < g->d; ++j) {
      const uint32_t t = stub(g, u, j);
      if (t == u) continue;
      __atomic_fetch_add(&g->deg[u], 1u, __ATOMIC_RELAXED);
      __atomic_fetch_add(&g->deg[t], 1u, __ATOMIC_RELAXED);
    }
}
static void pass_fill(void* p, uint64_t lo, uint64_t hi) {
  gen_ctx* g = p;
  for (uint64_t u = lo; u < hi; ++u)
    for (uint64_t j = 0; j < g->d; ++j) {
      const uint32_t t = stub(g, u, j);
      if (t == u) continue;
      g->slots[__atomic_fetch_add(&g->cur[u], 1ull, __ATOMIC_RELAXED)] = t;
      g->slots[__atomic_fetch_add(&g->cur[t], 1ull, __ATOMIC_RELAXED)] = (uint32_t)u;
    }
}
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}
static void pass_sort_unique(void* p, uint64_t lo, uint64_t hi) {
  gen_ctx* g = p;
  for (uint64_t v = lo; v < hi; ++v) {
    uint32_t* a = g->slots + g->off[v];
    const uint64_t len = g->off[v + 1] - g->off[v];
    if (len <= 32) { /* insertion sort */
      for (uint64_t i = 1; i < len; ++i) {
        const uint32_t x = a[i];
        uint64_t k = i;
        while (k > 0 && a[k - 1] > x) {
          a[k] = a[k - 1];
          --k;
        }
        a[k] = x;
      }
    } else {
      qsort(a, len, 4, cmp_u32);
    }
    uint64_t w = 0;
    for (uint64_t i = 0; i < len; ++i)
      if (i == 0 || a[i] != a[w - 1]) a[w++] = a[i];
    g->newdeg[v] = w;
  }
}
static void pass_copy(void* p, uint64_t lo, uint64_t hi) {
  gen_ctx* g = p;
  for (uint64_t v = lo; v < hi; ++v) memcpy(g->t + g->o[v], g->slots + g->off[v], g->newdeg[v] * 4);
}

int vp_synth_community_powerlaw(uint64_t n, uint64_t d, uint32_t C, double p_in, uint64_t seed,
                                unsigned threads, uint64_t** off_out, uint32_t** tgt_out,
                                uint64_t* m_out, uint32_t* labels) {
  return vp_synth_community_powerlaw_skew(n, d, C, p_in, 2.0, seed, threads, off_out, tgt_out, m_out, labels);
}

int vp_synth_community_powerlaw_skew(uint64_t n, uint64_t d, uint32_t C, double p_in, double skew, uint64_t seed,
                                     unsigned threads, uint64_t** off_out, uint32_t** tgt_out,
                                     uint64_t* m_out, uint32_t* labels) {
  if (!(skew >= 1.0 && skew <= 64.0)) return VP_PARAMETER;
  if (n < 2 || n > (1ull << 32) || d < 1 || C < 1 || C > n || !(p_in >= 0.0 && p_in <= 1.0))
    return VP_PARAMETER;
  gen_ctx g = {0};
  g.n = n;
  g.d = d;
  g.C = C;
  g.p_in = p_in;
  g.skew = skew;
  g.base_key = key_step(key_step(seed, 0xA1), 3);
  /* vertex placement: one seeded Fisher-Yates, stream (0xA1, 4) */
  g.rank_to_vertex = malloc(n * 4);
  g.vertex_to_rank = malloc(n * 4);
  for (uint64_t i = 0; i < n; ++i) g.rank_to_vertex[i] = (uint32_t)i;
  vp_stream rng;
  vp_stream_init(&rng, key_step(key_step(seed, 0xA1), 4));
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = vp_next_below(&rng, i);
    const uint32_t x = g.rank_to_vertex[i - 1];
    g.rank_to_vertex[i - 1] = g.rank_to_vertex[j];
    g.rank_to_vertex[j] = x;
  }
  for (uint64_t i = 0; i < n; ++i) g.vertex_to_rank[g.rank_to_vertex[i]] = (uint32_t)i;
  if (labels)
    for (uint64_t v = 0; v < n; ++v) labels[v] = comm_of_rank(&g, g.vertex_to_rank[v]);
  g.deg = calloc(n, 4);
  parallel_rows(threads, n, pass_degrees, &g);
  g.off = malloc((n + 1) * 8);
  g.off[0] = 0;
  for (uint64_t v = 0; v < n; ++v) g.off[v + 1] = g.off[v] + g.deg[v];
  free(g.deg);
  g.slots = malloc((g.off[n] ? g.off[n] : 1) * 4);
  g.cur = malloc(n * 8);
  memcpy(g.cur, g.off, n * 8);
  parallel_rows(threads, n, pass_fill, &g);
  free(g.cur);
  g.newdeg = malloc(n * 8);
  parallel_rows(threads, n, pass_sort_unique, &g);
  g.o = malloc((n + 1) * 8);
  g.o[0] = 0;
  for (uint64_t v = 0; v < n; ++v) g.o[v + 1] = g.o[v] + g.newdeg[v];
  const uint64_t m = g.o[n];
  g.t = malloc((m ? m : 1) * 4);
  parallel_rows(threads, n, pass_copy, &g);
  free(g.slots);
  free(g.off);
  free(g.newdeg);
  free(g.rank_to_vertex);
  free(g.vertex_to_rank);
  *off_out = g.o;
  *tgt_out = g.t;
  *m_out = m;
  return VP_OK;
}

/* ---------------------------------------------------------- feature rows */
typedef struct {
  uint64_t seed;
  uint32_t D;
  int fp16;
  void* out;
} feat_ctx;
static void pass_features(void* p, uint64_t lo, uint64_t hi) {
  feat_ctx* f = p;
  for (uint64_t v = lo; v < hi; ++v) {
    if (f->fp16)
      vp_features(f->seed, f->D, 1, (const uint32_t[]){(uint32_t)v}, 1, (uint16_t*)f->out + v * f->D);
    else
      vp_features(f->seed, f->D, 0, (const uint32_t[]){(uint32_t)v}, 1, (float*)f->out + v * f->D);
  }
}
void vp_fill_features(uint64_t seed, uint32_t D, int fp16, uint64_t n, void* out, unsigned threads) {
  feat_ctx f = {seed, D, fp16, out};
  parallel_rows(threads, n, pass_features, &f);
}

typedef struct {
  const unsigned char* table;
  uint64_t row_bytes;
  const uint32_t* ids;
  unsigned char* out;
} gather_ctx;
static void pass_gather(void* p, uint64_t lo, uint64_t hi) {
  gather_ctx* g = p;
  for (uint64_t i = lo; i < hi; ++i)
    memcpy(g->out + i * g->row_bytes, g->table + (uint64_t)g->ids[i] * g->row_bytes, g->row_bytes);
}
/* out[i, :] = table[ids[i], :] (the gather of SURVEY §8a A9) */
void vp_gather_rows(const void* table, uint64_t row_bytes, const uint32_t* ids, uint64_t count, void* out,
                    unsigned threads) {
  gather_ctx g = {table, row_bytes, ids, out};
  parallel_rows(threads, count, pass_gather, &g);
}
