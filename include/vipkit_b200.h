/*
 * vipkit_b200 — C ABI of the B200-native VIP-analysis + sample/gather hot path.
 *
 * This is the drop-in boundary. The reference (/root/reference/proj, "vipkit")
 * exposes the path as a C++20 API in namespace vipkit and has NO C ABI / FFI of
 * its own. Each entry point below names the reference interface it
 * replaces (file:line under /root/reference/proj). Plain pointers and sizes
 * only: no torch or C++ types cross this boundary. The C++ mirror of the
 * reference API (include/vipkit_b200/vipkit.hpp, namespace vipkit) and the
 * Python mirror (paper_2305_03152_b200/vipkit.py) are thin layers over it.
 *
 * Conventions
 *   - Every function returns a vk_status; VK_OK == 0. On failure a
 *     thread-local message is available from vk_last_error(). Codes 1..9 are
 *     the reference exception types (include/vipkit/error.hpp:8-38); the C++
 *     mirror rethrows them as those types.
 *   - "host" pointers are ordinary CPU memory owned by the caller; "_device"
 *     variants take device pointers owned by the caller and a cudaStream_t
 *     passed as void*. Device memory behind handles is owned by the handle.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with VK_ERR_CUDA.
 */
#ifndef VIPKIT_B200_H
#define VIPKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VK_API __attribute__((visibility("default")))
#else
#define VK_API
#endif

typedef enum vk_status {
  VK_OK = 0,
  VK_ERR_PARSE = 1,       /* vipkit::parse_error      (error.hpp:11-13) */
  VK_ERR_RANGE = 2,       /* vipkit::range_error      (error.hpp:14-16) */
  VK_ERR_PARAMETER = 3,   /* vipkit::parameter_error  (error.hpp:17-19) */
  VK_ERR_FORMAT = 4,      /* vipkit::format_error     (error.hpp:20-22) */
  VK_ERR_PARTITION = 5,   /* vipkit::partition_error  (error.hpp:23-25) */
  VK_ERR_SAMPLING = 6,    /* vipkit::sampling_error   (error.hpp:26-28) */
  VK_ERR_CONFIG = 7,      /* vipkit::config_error     (error.hpp:29-31) */
  VK_ERR_SHAPE = 8,       /* vipkit::shape_error      (error.hpp:32-34) */
  VK_ERR_IO = 9,          /* vipkit::io_error         (error.hpp:35-37) */
  VK_ERR_CUDA = 20,       /* CUDA runtime failure / no device */
                          /* 21: unused (the exchange is CUDA IPC + NVLink, no NCCL) */
  VK_ERR_UNSUPPORTED = 22,
  VK_ERR_INTERNAL = 23
} vk_status;

#define VK_MAX_HOPS 8
#define VK_MISS 0xFFFFFFFFu

typedef void* vk_stream_t; /* cudaStream_t */
typedef struct vk_graph_s* vk_graph;
typedef struct vk_sampler_s* vk_sampler;
typedef struct vk_plane_s* vk_plane;

/* ------------------------------------------------------------------ misc */
VK_API const char* vk_last_error(void);
VK_API const char* vk_status_name(int status);
VK_API int vk_version(void);
/* Number of sm_100 devices visible; 0 (and VK_OK) on a box without one. */
VK_API int vk_device_count(int* count);
VK_API int vk_device_alloc(int device, size_t bytes, void** out);
VK_API int vk_device_free(void* p);
/* Synchronous copy after draining all device work (plumbing for ctypes callers). */
VK_API int vk_memcpy(void* dst, const void* src, size_t bytes, int kind /*cudaMemcpyKind*/);
VK_API int vk_stream_sync(vk_stream_t stream);
/* Number of this library's kernels launched by the calling process so far
 * (bench.py reports the delta over the timed region as gpu_launches). */
VK_API uint64_t vk_launch_count(void);

/* ----------------------------------------------------------------- graph
 * Replaces vipkit::Graph (graph.hpp:20-46) + load_binary_csr (graph.hpp:117,
 * graph.cpp:565-598). Forward CSR: offsets u64[n+1], targets u32[m].
 * rev_* may be NULL: with VK_GRAPH_UNDIRECTED the reverse aliases the
 * forward structure (SPEC: undirected => rev == fwd); otherwise the reverse
 * CSR is built on the device by transposition (graph.cpp:587-595).
 * VK_GRAPH_VALIDATE runs check_invariants (graph.cpp:55-75) on the device
 * and fails with VK_ERR_FORMAT on violation. */
#define VK_GRAPH_UNDIRECTED 1u
#define VK_GRAPH_VALIDATE 2u
VK_API int vk_graph_create(int device, uint64_t n, uint64_t m, const uint64_t* fwd_offsets,
                           const uint32_t* fwd_targets, const uint64_t* rev_offsets,
                           const uint32_t* rev_targets, uint32_t flags, vk_graph* out);
/* VCSR file: "VCSR", u32 version 1, u64 n, u64 m, (n+1) u64 offsets, m u64
 * targets, little-endian (graph.hpp:113-117). Parsed on the host in parallel,
 * reverse built and invariants checked on the device. */
VK_API int vk_graph_load_vcsr(int device, const char* path, uint32_t flags, vk_graph* out);
VK_API int vk_graph_destroy(vk_graph g);
VK_API int vk_graph_info(vk_graph g, uint64_t* n, uint64_t* m, int* symmetric, int* device);
VK_API int vk_graph_copy_forward(vk_graph g, uint64_t* fwd_offsets, uint32_t* fwd_targets);
/* vipkit::apply_reorder's graph part (reorder.hpp:34-35, reorder.cpp:36-70):
 * a new device graph whose vertex u is old vertex old_of_new[u] (n entries,
 * host), every neighbour list relabelled through the inverse map and sorted
 * ascending, reverse CSR rebuilt. Roles and labels permute on the host
 * (role'[u] = role[old_of_new[u]]). VK_ERR_SHAPE if the map is not a
 * permutation. */
VK_API int vk_graph_apply_reorder(vk_graph g, const uint32_t* old_of_new, vk_graph* out);
VK_API int vk_graph_copy_reverse(vk_graph g, uint64_t* rev_offsets, uint32_t* rev_targets);

/* ------------------------------------------------------------------- VIP
 * vipkit::initial_probs (vip.hpp:39-40, vip.cpp:25-35). Host arrays.
 * roles: u8 codes (0 = train, graph.hpp:48). */
VK_API int vk_initial_probs(uint64_t n, const uint8_t* roles, const uint32_t* part_of, uint32_t k,
                            uint64_t batch_size, double* p0_out);
/* vipkit::propagate (vip.hpp:45-46, vip.cpp:37-83) for `ncols` independent p0
 * vectors at once (e.g. all K partitions: one pass over the reverse CSR
 * serves every column). p0: ncols x n (column c = vector c, contiguous).
 * hop_out: ncols x L x n or NULL; total_out: ncols x n. Host buffers. */
/* Storage width of the hoisted log terms between hops (process-wide): 0 =
 * automatic (double while n x columns x 8 B fits 64 MB, else float with a
 * guarded fallback to double), 32 or 64 to force one (tests). */
VK_API int vk_vip_force_storage(int bits);
VK_API int vk_vip_propagate(vk_graph g, const uint32_t* fanouts, uint32_t num_hops,
                            uint32_t ncols, const double* p0, double* hop_out, double* total_out);
/* Same on device buffers, asynchronous on `stream`. */
VK_API int vk_vip_propagate_device(vk_graph g, const uint32_t* fanouts, uint32_t num_hops,
                                   uint32_t ncols, const double* p0_dev, double* hop_dev,
                                   double* total_dev, vk_stream_t stream);

/* -------------------------------------------------------------- sampling
 * vipkit::epoch_minibatches (sampling.hpp:43-47, sampling.cpp:45-70): the
 * seeded permutation of partition-k train vertices (host; one sequential
 * Fisher-Yates stream per (epoch, k)). Batches are the consecutive b-chunks of
 * out_perm (capacity n); *out_count = |T_k|. seed_keys may be NULL. */
VK_API int vk_epoch_minibatches(uint64_t n, const uint8_t* roles, const uint32_t* part_of,
                                uint32_t k, uint64_t batch_size, uint64_t epoch,
                                uint64_t global_seed, const uint32_t* seed_keys,
                                uint32_t* out_perm, uint64_t* out_count);

/* PartitionMap::train_members (graph.hpp:68, graph.cpp:106-111): the train
 * vertices of partition k in ascending id order (out capacity n). */
VK_API int vk_train_members(uint64_t n, const uint8_t* roles, const uint32_t* part_of, uint32_t k,
                            uint32_t* out, uint64_t* out_count);
/* The shuffle half of epoch_minibatches (sampling.cpp:54-63) over a train
 * member list computed once (vk_train_members): out = the epoch-e
 * permutation, identical to vk_epoch_minibatches' for seed_keys = NULL. out
 * may alias train. Empty lists raise VK_ERR_SAMPLING (sampling.cpp:50-53). */
VK_API int vk_epoch_shuffle(const uint32_t* train, uint64_t count, uint32_t k, uint64_t epoch,
                            uint64_t global_seed, uint32_t* out);

/* vipkit::sample_neighbors (sampling.hpp:54-56, sampling.cpp:72-92) for one
 * vertex on the device: appends min(fanout, deg v) ids to out (capacity
 * fanout); *stream_state is RngStream's counter, advanced by the draws as the
 * reference's stream is. neighbor_keys (deg(v) host entries in CSR row order,
 * the seed_keys of v's neighbours) or NULL: with keys the draws run over the
 * row ordered by key (sampling.cpp:83-85). */
VK_API int vk_graph_sample_neighbors(vk_graph g, uint32_t v, uint32_t fanout, uint64_t* stream_state,
                                     const uint32_t* neighbor_keys, uint32_t* out, uint64_t* out_count);

/* vipkit::BatchRef (sampling.hpp:33-37). */
typedef struct vk_batch_ref {
  uint64_t epoch;
  uint64_t batch_index;
  uint32_t partition;
  uint32_t reserved;
} vk_batch_ref;

typedef struct vk_sampler_config {
  uint32_t num_hops;                /* L = FanoutSpec::hops() */
  uint32_t fanouts[VK_MAX_HOPS];    /* FanoutSpec::fanouts (sampling.hpp:14-21) */
  uint64_t batch_size;              /* max seeds per minibatch (b) */
  uint32_t max_minibatches;         /* minibatches per wave (device batching) */
  uint32_t flags;                   /* VK_SAMPLER_* frontier representation, 0 = automatic */
  uint64_t global_seed;             /* SeedSpec::global_seed (rng.hpp:59) */
} vk_sampler_config;

/* Frontier representation (results are identical): dense = n-bit bitmaps per
 * minibatch (graphs where a frontier covers a sizeable fraction of n), sparse
 * = vertex-range buckets deduplicated in shared memory (papers-scale graphs).
 * Automatic: sparse when n >= 16 x the per-minibatch vertex capacity. */
#define VK_SAMPLER_FORCE_DENSE 1u
#define VK_SAMPLER_FORCE_SPARSE 2u
VK_API int vk_sampler_create(vk_graph g, const vk_sampler_config* cfg, vk_sampler* out);
VK_API int vk_sampler_destroy(vk_sampler s);
/* seed_keys replay (sampling.hpp:43-64, `seed_keys` of expand /
 * sample_neighbors): vertex v's stream is keyed by seed_keys[v] instead of v
 * and a partial Fisher-Yates draws from v's neighbours ordered by their keys
 * (sampling.cpp:83-85, 108-112), so expansions of a relabelled graph replay
 * the original graph's (with seed_keys = old_of_new). seed_keys: n entries,
 * distinct within every neighbour list (a relabelling); NULL turns replay off.
 * Batches given to vk_sampler_run are taken as is (order them with
 * vk_epoch_minibatches' seed_keys). */
VK_API int vk_sampler_set_seed_keys(vk_sampler s, const uint32_t* seed_keys);
/* vipkit::expand (sampling.hpp:62-64, sampling.cpp:94-128) for a wave of
 * `nmb` minibatches: per hop h, every vertex of F_{h-1} draws with stream
 * (0xB2, epoch, partition, batch_index, h, v) -> bit-identical frontiers
 * F_1..F_L (sorted, distinct), all_vertices (sorted distinct union), the MFG
 * edge list and the relabel maps. seeds: concatenated batches, minibatch i =
 * seeds[seed_offsets[i] .. seed_offsets[i+1]) (seed_offsets is host memory);
 * seeds is a host pointer unless seeds_on_device. Asynchronous on `stream`
 * (NULL = the sampler's own stream). Outputs stay on the device until the
 * next run. Errors: VK_ERR_SAMPLING for an empty batch (sampling.cpp:97). */
VK_API int vk_sampler_run(vk_sampler s, uint32_t nmb, const vk_batch_ref* refs,
                          const uint32_t* seeds, const uint64_t* seed_offsets,
                          int seeds_on_device, vk_stream_t stream);
/* Sizes of the last run (synchronises): frontier_sizes[nmb*L] = |F_h|,
 * edge_counts[nmb*L] = MFG edges of hop h, all_sizes[nmb] = |all_vertices|.
 * Any pointer may be NULL. */
VK_API int vk_sampler_sizes(vk_sampler s, uint64_t* frontier_sizes, uint64_t* edge_counts,
                            uint64_t* all_sizes);
/* Host copies of one minibatch's outputs from the last run (synchronous).
 * hop is 1-based for frontiers/MFG; relabel hop 0 is the batch. */
VK_API int vk_sampler_copy_frontier(vk_sampler s, uint32_t mb, uint32_t hop, uint32_t* out);
VK_API int vk_sampler_copy_all(vk_sampler s, uint32_t mb, uint32_t* out);
/* MFG of hop h: indptr[|F_{h-1}|+1] (u64 edge offsets per source, sources in
 * expand's visiting order) and dst[edges] = index of the sampled vertex in
 * F_h (the relabelled edge list; the global id is F_h[dst]). */
VK_API int vk_sampler_copy_mfg(vk_sampler s, uint32_t mb, uint32_t hop, uint64_t* indptr,
                               uint32_t* dst);
/* Relabel map: all_index[i] = position of F_hop[i] in all_vertices. */
VK_API int vk_sampler_copy_relabel(vk_sampler s, uint32_t mb, uint32_t hop, uint32_t* all_index);

/* Device views of the last run (for downstream kernels / the GNN). Region of
 * minibatch i = base + i * stride (elements). Counts are device u32 arrays. */
typedef struct vk_sampler_view {
  uint32_t nmb, num_hops;
  const uint32_t* all;            uint64_t all_stride;      const uint32_t* all_count;
  const uint32_t* frontier[VK_MAX_HOPS + 1]; uint64_t frontier_stride[VK_MAX_HOPS + 1];
  const uint32_t* frontier_count[VK_MAX_HOPS + 1];          /* [0] = batch */
  const uint32_t* mfg_indptr[VK_MAX_HOPS + 1];              /* u32 offsets, [h] for hop h */
  const uint32_t* mfg_dst[VK_MAX_HOPS + 1]; uint64_t mfg_stride[VK_MAX_HOPS + 1];
  const uint32_t* all_index[VK_MAX_HOPS + 1];               /* stride = frontier_stride */
} vk_sampler_view;
VK_API int vk_sampler_get_view(vk_sampler s, vk_sampler_view* view);
/* Asynchronous device-to-device snapshot of the last run's count block
 * (u32: |F_h| [(L+1) x max_mb] | MFG edges [(L+1) x max_mb] | |all| [max_mb]
 * | error flag) into dst_dev; *words receives its length. Lets a caller keep
 * per-wave sizes without a host synchronisation. */
VK_API int vk_sampler_snapshot_counts(vk_sampler s, uint32_t* dst_dev, uint64_t* words,
                                      vk_stream_t stream);

/* Device-side RngStream draws (rng.hpp:19-44) for conformance tests:
 * `count` values of next_below(bound) (next_u64 when bound == 0). */
VK_API int vk_debug_stream_draws(int device, uint64_t key, uint64_t bound, uint64_t count,
                                 uint64_t* out);

/* --------------------------------------------------- ranking / cache plan
 * vipkit::rank_by_scores -> order_remotes (policies.hpp:48, policies.cpp:
 * 20-34, 134-138): vertices with part_of != k ordered by (score desc, id asc),
 * computed by a device radix sort. order_out/score_out capacity n. */
VK_API int vk_rank_by_scores(int device, uint64_t n, const uint32_t* part_of, uint32_t k,
                             const double* scores, uint64_t n_scores, uint32_t* order_out,
                             double* score_out, uint64_t* count_out);
/* Baseline rankings of the Fig. 3 sweep (policies.hpp:24-45, policies.cpp:
 * 57-132), scores computed on the device, remotes ordered as order_remotes.
 * Bit-identical to the reference (sequential in-neighbour sums in CSR order,
 * round-to-nearest f64).
 *  - rank_degree: remotes reachable within L forward hops of partition k's
 *    train vertices first, by decreasing out-degree; unreachable score 0.
 *  - rank_halo_1hop: remote out-neighbours of partition k (score 1);
 *    *effective_alpha = |halo| * K / n (may be NULL).
 *  - rank_wpr: weighted reverse PageRank, restart uniform over k's train
 *    vertices, hop-1 weights of TransitionModel{hop1_fanout}, `iters` power
 *    steps with `damping` (reference defaults 5, 0.85).
 *  - rank_numpaths: walks of length <= L from k's train vertices (f64). */
VK_API int vk_rank_degree(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                          uint32_t L, uint32_t* order_out, double* score_out, uint64_t* count_out);
VK_API int vk_rank_halo_1hop(vk_graph g, const uint32_t* part_of, uint32_t K, uint32_t k, uint32_t* order_out,
                             double* score_out, uint64_t* count_out, double* effective_alpha);
VK_API int vk_rank_wpr(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                       uint32_t hop1_fanout, uint32_t iters, double damping, uint32_t* order_out,
                       double* score_out, uint64_t* count_out);
VK_API int vk_rank_numpaths(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                            uint32_t L, uint32_t* order_out, double* score_out, uint64_t* count_out);
/* build_cache capacity (policies.cpp:155-156): floor(alpha*n/K + 1e-9). */
VK_API int vk_cache_capacity(double alpha, uint64_t n, uint32_t K, uint64_t* capacity);
/* vipkit::build_reorder (reorder.hpp:25-26, reorder.cpp:11-34) on the device:
 * partition-contiguous ranges, each ordered by (score_k desc, id asc).
 * scores: K x n. ranges: 2K u64 [start, end). */
VK_API int vk_build_reorder(int device, uint64_t n, uint32_t K, const uint32_t* part_of,
                            const double* scores, uint32_t* old_of_new, uint64_t* ranges);

/* ------------------------------------------------------ feature plane
 * The VIP-ordered feature store (north-star (3); no reference code: features
 * are never materialised there). For each partition k resident
 * on this device: local rows = members of k in build_reorder order, then
 * cache rows = the CachePlan prefix of ranking k (policies.cpp:149-163) in
 * ascending vertex id, and a cache index (membership bits + rank per 64 ids).
 * Rows are `dim` values
 * of dtype VK_F32 or VK_F16. Partitions owned by another GPU are attached by
 * CUDA IPC and read over NVLink inside the gather kernel. */
#define VK_F32 0
#define VK_F16 1
VK_API int vk_plane_create(int device, uint64_t n, uint32_t K, uint32_t dim, int dtype,
                           const uint32_t* part_of, const uint32_t* old_of_new,
                           const uint64_t* ranges, vk_plane* out);
VK_API int vk_plane_destroy(vk_plane p);
/* Make partition k resident: local rows + cache rows (cache_ids in ranking
 * order, n_cache of them). features: host n x dim rows in global-id order, or
 * NULL to synthesise rows on the device from `feature_seed` (the generator of
 * SURVEY §8d, identical to oracle vp_feature_*). */
VK_API int vk_plane_load_partition(vk_plane p, uint32_t k, const uint32_t* cache_ids,
                                   uint64_t n_cache, const void* features, uint64_t feature_seed);
/* CachePlan::is_cached (policies.hpp:58-60). */
VK_API int vk_plane_is_cached(vk_plane p, uint32_t k, uint32_t v, int* out);
/* CUDA IPC export of partition k's local rows (64-byte handle) and import of
 * a peer's (multi-GPU: one process per GPU). */
VK_API int vk_plane_export(vk_plane p, uint32_t k, void* handle64, uint64_t* rows);
VK_API int vk_plane_attach(vk_plane p, uint32_t k, const void* handle64, uint64_t rows);
/* classify (commsim.cpp:61-73) + gather for every minibatch of the sampler's
 * last run: out[i][r][:] = X[all_vertices_i[r]][:] (out region i starts at
 * out + i*out_stride_rows*row_bytes), from the local rows, the cache rows or
 * (miss) the owner partition's rows -- local HBM or a peer over NVLink.
 * counts_dev (device u64, nmb x 4, zeroed by the call): local, cache, miss,
 * miss rows served from another GPU. With attached peer partitions the wave's
 * remote misses are first deduplicated (union over all minibatches of the
 * wave) and each distinct row is pulled once over NVLink into local staging
 * (the miss exchange); the rows are then copied from there. Asynchronous on
 * `stream`. */
VK_API int vk_plane_gather(vk_plane p, vk_sampler s, void* out_dev, uint64_t out_stride_rows,
                           uint64_t* counts_dev, vk_stream_t stream);
VK_API int vk_plane_row_bytes(vk_plane p, uint64_t* row_bytes);
/* Multi-GPU: issue the miss exchange (remote-miss union, NVLink pull into
 * staging) of sampler s's last run now, on the plane's auxiliary stream
 * (after the sampler's work), so it overlaps whatever the caller queues next
 * (e.g. the next wave's vk_sampler_run on a second sampler); the following
 * vk_plane_gather of that run waits for it instead of exchanging again.
 * No-op without attached peer partitions. */
VK_API int vk_plane_prefetch(vk_plane p, vk_sampler s);
/* vk_plane_prefetch ordered after the work queued so far on `after` as well
 * (e.g. the gather of the previous wave), so the NVLink pull overlaps the
 * next wave's latency-bound sampling instead of contending with an
 * HBM-bound gather. */
VK_API int vk_plane_prefetch_after(vk_plane p, vk_sampler s, vk_stream_t after);
/* Distinct remote rows the last multi-GPU gather pulled over NVLink (the
 * wave's deduplicated miss exchange); synchronises the device. */
VK_API int vk_plane_pulled_rows(vk_plane p, uint64_t* rows);

/* ------------------------------------------------ communication tallies
 * vipkit::simulate (commsim.hpp:56-59, commsim.cpp:77-127) and the alpha
 * axis of sweep (commsim.cpp:140-259): expands every minibatch
 * of every partition for `epochs` epochs in for_each_expansion order
 * (commsim.cpp:45-52) with the device sampler (waves of `wave` minibatches,
 * 0 = 128) and classifies each distinct neighbourhood vertex of a minibatch
 * of partition k as local / cache hit / remote miss (commsim.cpp:61-73).
 * Cache plans: partition k's cached ids are cached_ids[cached_offsets[k] ..
 * cached_offsets[k+1]) in ranking order; plan a caches the first
 * takes[a*K + k] of them (build_cache's ranking prefixes), takes == NULL
 * means one plan caching every listed id. seed_keys (n entries or NULL) is
 * SimulateOptions::seed_keys: replay streams keyed by e.g. original ids
 * (vk_sampler_set_seed_keys). cells[num_plans][epochs][K][3] =
 * {local_hits, cache_hits, remote_misses} (CommReport::Cell). Errors as the
 * reference: VK_ERR_SAMPLING for a partition without train vertices,
 * VK_ERR_PARAMETER for batch_size 0. */
VK_API int vk_simulate(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K,
                       const uint32_t* fanouts, uint32_t num_hops, uint64_t batch_size, uint64_t epochs,
                       uint64_t global_seed, const uint32_t* seed_keys, const uint32_t* cached_ids,
                       const uint64_t* cached_offsets,
                       const uint64_t* takes, uint32_t num_plans, uint32_t wave, uint64_t* cells);
/* vk_simulate for one plan (cached ids as above, takes = NULL) with the
 * per-minibatch rows of SimulateOptions::batch_costs (commsim.hpp:42-51,
 * commsim.cpp:104-118): batch_rows[i*7..] = {epoch, batch_index, partition,
 * local - gpu, gpu, cache, miss} for the i-th minibatch in for_each_expansion
 * order; gpu counts local vertices whose position in gpu_orderings[k]
 * (gpu_ordering_sizes[k] ids) is below floor(gamma*size + 1e-9), 0 without
 * orderings. *num_batches = the minibatch count (batch_rows may be NULL to
 * query it; else capacity >= count or VK_ERR_SHAPE). */
VK_API int vk_simulate_batches(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K,
                               const uint32_t* fanouts, uint32_t num_hops, uint64_t batch_size, uint64_t epochs,
                               uint64_t global_seed, const uint32_t* seed_keys, const uint32_t* cached_ids,
                               const uint64_t* cached_offsets, const uint32_t* const* gpu_orderings,
                               const uint64_t* gpu_ordering_sizes, double gamma, uint64_t* cells,
                               uint64_t* batch_rows, uint64_t batch_rows_capacity, uint64_t* num_batches);
/* The "oracle" policy's retrospective access counts (sweep pass 1,
 * commsim.cpp:155-166): counts[k*n + v] = minibatches of partition k over
 * `epochs` epochs (for_each_expansion order) whose all_vertices contain v. */
VK_API int vk_access_counts(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K,
                            const uint32_t* fanouts, uint32_t num_hops, uint64_t batch_size, uint64_t epochs,
                            uint64_t global_seed, double* counts);
/* vipkit::empirical_vip (vip.hpp:52-55, vip.cpp:85-105), the "sim." policy's
 * estimate: S epochs of partition k's minibatches under
 * SeedSpec::derived(0xC1) through the device sampler; freq[v] = (number of
 * minibatches whose all_vertices contain v) / (number of minibatches).
 * Bit-identical to the reference. VK_ERR_PARAMETER for S = 0. */
VK_API int vk_empirical_vip(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                            uint64_t batch_size, const uint32_t* fanouts, uint32_t num_hops, uint64_t epochs,
                            uint64_t global_seed, double* freq);

/* ------------------------------------------------------- synthetic data
 * Community-structured power-law generator for the BASELINE configs (builder
 * addition: the reference PA generator is sequential and
 * has no partitionable structure). Deterministic for any thread count:
 * every stub (u, j) draws from its own counter-keyed stream. Output is an
 * undirected, deduplicated, self-loop-free CSR (graph.hpp:17-19 invariants);
 * community labels (u32[n], C communities, balanced) double as partition
 * labels. The caller frees the returned arrays with vk_host_free. */
VK_API int vk_synth_community_powerlaw(uint64_t n, uint64_t d, uint32_t communities,
                                       double p_in, uint64_t seed, unsigned threads,
                                       uint64_t** offsets, uint32_t** targets, uint64_t* m,
                                       uint32_t* labels);
/* ... with the popularity skew as a parameter: the target is the member of
 * popularity rank floor(size * U^skew) (skew 2 above; larger concentrates
 * the edges on fewer, bigger hubs). */
VK_API int vk_synth_community_powerlaw_skew(uint64_t n, uint64_t d, uint32_t communities, double p_in,
                                            double skew, uint64_t seed, unsigned threads, uint64_t** offsets,
                                            uint32_t** targets, uint64_t* m_out, uint32_t* labels);
/* vipkit::make_roles (graph.hpp:93-94, graph.cpp:247-268). */
VK_API int vk_synth_roles(uint64_t n, double train, double valid, double test, uint64_t seed,
                          uint8_t* roles);
VK_API void vk_host_free(void* p);

/* ------------------------------------------------------------ file formats
 * (csrc/io.cu) Text files: one decimal value per line, empty and '#' lines
 * skipped, a line's leading digits are its value (std::from_chars), anything
 * else VK_ERR_FORMAT naming file:line; unopenable files VK_ERR_IO.
 * partition_from_file (graph.hpp:105, graph.cpp:461-484): exactly n labels,
 * K == 0 infers max+1 (*K_out), then PartitionMap::from_labels' checks
 * (label >= K: VK_ERR_FORMAT, empty partition: VK_ERR_PARTITION). */
VK_API int vk_partition_from_file(const char* path, uint32_t K, uint64_t n, uint32_t* part_of,
                                  uint32_t* K_out);
/* write_partition_labels (graph.hpp:122, graph.cpp:624-628) */
VK_API int vk_write_partition_labels(const char* path, const uint32_t* part_of, uint64_t n);
/* load_roles (graph.hpp:119, graph.cpp:600-616): codes 0..3; *roles is
 * allocated (vk_host_free). write_roles (graph.hpp:120, graph.cpp:618-622). */
VK_API int vk_load_roles(const char* path, uint8_t** roles, uint64_t* n);
VK_API int vk_write_roles(const char* path, const uint8_t* roles, uint64_t n);
/* write_vip_binary / load_vip_binary (vip.hpp:58-59, vip.cpp:107-134): n
 * little-endian f64 totals; *values allocated (vk_host_free). */
VK_API int vk_write_vip_binary(const char* path, const double* total, uint64_t n);
VK_API int vk_load_vip_binary(const char* path, double** values, uint64_t* n);
/* write_binary_csr (graph.hpp:116, graph.cpp:553-563): the VCSR file
 * vk_graph_load_vcsr reads. */
VK_API int vk_write_vcsr(const char* path, uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt);

#ifdef __cplusplus
}
#endif
#endif /* VIPKIT_B200_H */
