/* TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * Plain-C restatement of the reference hot path (/root/reference/proj). It is
 * the CPU checker for the CUDA library and is never linked into the product.
 * Parity pinned against the compiled reference (_ref) and tests/golden.
 */
#ifndef VIPKIT_PORT_H
#define VIPKIT_PORT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same numbering as include/vipkit_b200.h */
enum { VP_OK = 0, VP_PARAMETER = 3, VP_FORMAT = 4, VP_PARTITION = 5, VP_SAMPLING = 6, VP_SHAPE = 8 };
const char* vp_last_error(void);

/* ---- rng (rng.hpp) ---- */
uint64_t vp_mix64(uint64_t x);
typedef struct { uint64_t counter; } vp_stream;
void vp_stream_init(vp_stream* s, uint64_t key);
uint64_t vp_next_u64(vp_stream* s);
double vp_next_double(vp_stream* s);
uint64_t vp_next_below(vp_stream* s, uint64_t bound);
uint64_t vp_seed_key(uint64_t seed, const uint64_t* parts, uint32_t np);
uint64_t vp_seed_derived(uint64_t seed, uint64_t tag);
void vp_stream_draws(uint64_t key, uint64_t bound, uint64_t count, uint64_t* out);

/* ---- graph (graph.cpp) ---- kinds follow SynthKind order (graph.hpp:80) */
enum { VP_PATH = 0, VP_STAR = 1, VP_TREE = 2, VP_GRID = 3, VP_PA = 4, VP_UNIFORM = 5 };
int vp_graph_from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst, uint64_t ne,
                        int undirected, uint64_t** off, uint32_t** tgt, uint64_t* m);
int vp_generate(int kind, uint64_t n, uint64_t d, uint64_t seed, uint64_t** off, uint32_t** tgt,
                uint64_t* m);
void vp_free(void* p);
int vp_make_roles(uint64_t n, double train, double valid, double test, uint64_t seed, uint8_t* out);

/* ---- sampling (sampling.cpp) ---- */
int vp_epoch_minibatches(const uint8_t* roles, uint64_t n, const uint32_t* labels, uint32_t k,
                         uint64_t b, uint64_t epoch, uint64_t seed, uint32_t* out_perm,
                         uint64_t* out_count);
uint64_t vp_sample_neighbors(const uint64_t* off, const uint32_t* tgt, uint32_t v, uint32_t fanout,
                             vp_stream* s, uint32_t* out);

typedef struct vp_expansion {
  uint32_t L;
  uint64_t nb;
  uint32_t* batch;
  uint64_t* fsize;     /* [L] */
  uint32_t** frontier; /* [L][fsize] sorted unique */
  uint64_t** indptr;   /* [L][|F_{h-1}|+1] MFG row pointers */
  uint32_t** edges;    /* [L][indptr[last]] sampled ids in draw order */
  uint64_t nall;
  uint32_t* all;       /* sorted unique union */
} vp_expansion;
vp_expansion* vp_expand(const uint64_t* off, const uint32_t* tgt, uint64_t n, const uint32_t* batch,
                        uint64_t nb, const uint32_t* fanouts, uint32_t L, uint64_t seed,
                        uint64_t epoch, uint32_t part, uint64_t batch_index);
void vp_expansion_free(vp_expansion* x);

/* ---- vip (vip.cpp) ---- */
int vp_initial_probs(const uint8_t* roles, uint64_t n, const uint32_t* labels, uint32_t k,
                     uint64_t b, double* out);
int vp_propagate(const uint64_t* fwd_off, const uint64_t* rev_off, const uint32_t* rev_tgt,
                 uint64_t n, const uint32_t* fanouts, uint32_t L, const double* p0,
                 double* hop_out /* L*n or NULL */, double* total_out);

/* ---- policies (policies.cpp) / commsim (commsim.cpp) / reorder (reorder.cpp) ---- */
int vp_rank_by_scores(const uint32_t* labels, uint64_t n, uint32_t k, const double* scores,
                      uint32_t* order_out, double* score_out, uint64_t* count);
int vp_cache_capacity(double alpha, uint64_t n, uint32_t K, uint64_t* cap);
void vp_classify(const uint32_t* all, uint64_t nall, const uint32_t* labels, uint32_t k,
                 const uint64_t* cache_bits, uint64_t counts[3]);
int vp_build_reorder(const uint32_t* labels, uint64_t n, uint32_t K, const double* scores,
                     uint32_t* old_of_new, uint64_t* ranges);

/* ---- synthetic feature rows (builder contract) ---- */
float vp_feature_f32(uint64_t seed, uint64_t v, uint32_t j, uint32_t D);
uint16_t vp_feature_f16_bits(uint64_t seed, uint64_t v, uint32_t j, uint32_t D);
void vp_features(uint64_t seed, uint32_t D, int fp16, const uint32_t* ids, uint64_t count,
                 void* out);


/* ---- workload (workload.c): bench graph recipe, feature table, CPU gather ---- */
int vp_synth_community_powerlaw(uint64_t n, uint64_t d, uint32_t C, double p_in, uint64_t seed,
                                unsigned threads, uint64_t** off_out, uint32_t** tgt_out,
                                uint64_t* m_out, uint32_t* labels);
int vp_synth_community_powerlaw_skew(uint64_t n, uint64_t d, uint32_t C, double p_in, double skew, uint64_t seed,
                                     unsigned threads, uint64_t** off_out, uint32_t** tgt_out,
                                     uint64_t* m_out, uint32_t* labels);
void vp_fill_features(uint64_t seed, uint32_t D, int fp16, uint64_t n, void* out, unsigned threads);
void vp_gather_rows(const void* table, uint64_t row_bytes, const uint32_t* ids, uint64_t count, void* out,
                    unsigned threads);

#ifdef __cplusplus
}
#endif
#endif
