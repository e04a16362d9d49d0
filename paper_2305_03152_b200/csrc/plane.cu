// Ranking, cache plan and the VIP-ordered feature plane with the fused
// classify + gather kernel.
//
//  * vk_rank_by_scores   = order_remotes (/root/reference/proj/src/policies.cpp:
//    20-34, 134-138) as a stable device radix sort on an order-preserving key
//    of (score desc) over ids in ascending order -> ties by ascending id.
//  * vk_build_reorder    = build_reorder (reorder.cpp:11-34): two stable sorts
//    (score desc within partition, then partition id).
//  * feature plane       = the north-star's VIP-ordered store: per resident
//    partition k, local rows in build_reorder order then the cache rows (the
//    CachePlan prefix, policies.cpp:149-163) in ascending vertex id, plus a
//    cache index of one 16-byte word per 64 vertex ids (membership bits and
//    the cache rank of the word's first member).
//  * vk_plane_gather     = classify (commsim.cpp:61-73) + row gather for a
//    whole wave: 128-bit loads/stores, flattened over (row, 16-byte chunk) so
//    every lane moves data and writes are fully coalesced; misses read the
//    owner partition's rows from local HBM or, multi-GPU, from a staging
//    buffer filled by the wave's deduplicated miss exchange (remote-miss
//    union -> one NVLink pull per distinct row from the owner's HBM through
//    a CUDA IPC mapping), optionally issued early by vk_plane_prefetch.
#include <cub/cub.cuh>

#include <cmath>
#include <map>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "rng.cuh"
#include "scan.cuh"

struct vk_sampler_s;
namespace vk {
void sampler_internal(vk_sampler_s* s, const std::uint32_t** all, std::uint64_t* all_stride,
                      const std::uint32_t** all_count, std::uint32_t* nmb, const std::uint32_t** partitions,
                      vk_graph_s** g, cudaStream_t* last_stream);
std::uint64_t sampler_desc_stride();
void sampler_all_rank(vk_sampler_s* s, const uint4** rank, std::uint64_t* W);
bool sampler_all_rank_dense(vk_sampler_s* s);
const std::uint32_t* sampler_tile_base(vk_sampler_s* s, std::uint32_t* bucket_bits, std::uint32_t* nb);
std::uint64_t sampler_run_id(vk_sampler_s* s);
void sampler_host_partitions(vk_sampler_s* s, std::vector<std::uint32_t>& out);
cudaEvent_t sampler_done_event(vk_sampler_s* s);
void sampler_add_reader(vk_sampler_s* s, cudaStream_t st);
}  // namespace vk

struct vk_plane_s {
  int device = 0;
  std::uint64_t n = 0;
  std::uint32_t K = 0, dim = 0;
  int dtype = VK_F32;
  std::uint64_t row_bytes = 0;
  vk::DevBuf part_of, owner_row;  // u32 [n] each
  vk::DevBuf new_id;              // u32 [n]: reorder position (global row order)
  vk::DevBuf d_rstart;            // u32 [K+1]: partition range starts in row order
  std::vector<std::uint64_t> rstart, rend;
  std::vector<std::uint32_t> old_of_new;  // host copy (local row order)
  struct Part {
    bool resident = false, attached = false;
    vk::DevBuf store;  // (n_local + n_cache) rows
    vk::DevBuf cword;  // uint4 [W]: {member bits lo, hi, cache rank of the word's first member, 0}
    std::uint64_t n_local = 0, n_cache = 0;
    std::vector<std::uint64_t> cache_bits;  // CachePlan::member_bits[k]
    void* peer = nullptr;                   // IPC-mapped local rows of a remote partition
    vk::DevBuf rmask;  // [W] bit v: v is neither local nor cached here and its owner is on a peer GPU
  };
  std::vector<Part> parts;
  vk::DevBuf d_base, d_cword, d_nlocal;  // K-entry tables for the gather kernel
  vk::DevBuf d_rmask;                   // [K] Part::rmask pointers (resident partitions)
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;  // prefetched miss exchanges (vk_plane_prefetch), high priority
  cudaEvent_t after_ev = nullptr;  // vk_plane_prefetch_after ordering
  // per-wave deduplicated pull of remote rows (multi-GPU): union bitmap of
  // the wave's remote misses, its rank prefix, the distinct list, and the
  // local staging copy of those rows
  struct StageSet {
    vk::DevBuf ubits, uprefix, ulist, staging, scan_tmp;
    vk::DevBuf vbits;  // vertex-space union (word mark); cleared as consumed
    std::uint64_t stage_cap = 0;  // rows the staging buffer holds
    // vk_plane_prefetch: the exchange of sampler run `prefetched` was issued
    // on the aux stream and completes at `ready`
    std::uint64_t prefetched = ~0ull;
    cudaEvent_t ready = nullptr;
    ~StageSet() {
      if (ready) cudaEventDestroy(ready);
    }
  };
  // one set per sampler, so overlapped waves (one sampler per pipeline
  // stream) never share staging
  std::map<const void*, StageSet> stage_sets;
  const StageSet* last_set = nullptr;
};

namespace vk {
namespace {

// In-place exclusive scan of n u32 (scan.cuh); `tmp` holds the look-back status.
void exclusive_scan_u32(std::uint32_t* a, std::uint64_t n, DevBuf& tmp, cudaStream_t st) {
  const std::uint64_t tiles = ceil_div(n, (std::uint64_t)kScanU32Threads * kScanU32Items);
  if (tmp.bytes < tiles * 8) tmp.alloc(tiles * 8);
  VK_CUDA(cudaMemsetAsync(tmp.p, 0, tiles * 8, st));
  k_scan_u32<<<(unsigned)tiles, kScanU32Threads, 0, st>>>(a, n, tmp.as<unsigned long long>());
  VK_LAUNCH_CHECK();
}

// Order-preserving u64 key of a double, descending: -0.0 == +0.0 as in the
// reference comparator (policies.cpp:28).
__device__ __forceinline__ std::uint64_t desc_key(double x) {
  std::uint64_t b = (x == 0.0) ? 0ull : (std::uint64_t)__double_as_longlong(x);
  const std::uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;
}

__global__ void k_rank_keys(const double* __restrict__ scores, const std::uint32_t* __restrict__ part_of,
                            std::uint64_t n, std::uint32_t k, std::uint64_t* __restrict__ keys,
                            std::uint32_t* __restrict__ ids, unsigned long long* __restrict__ nremote) {
  std::uint64_t cnt = 0;
  for (std::uint64_t v = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (std::uint64_t)gridDim.x * blockDim.x) {
    const bool remote = part_of[v] != k;
    keys[v] = remote ? desc_key(scores[v]) : ~0ull;  // locals sort to the tail
    ids[v] = (std::uint32_t)v;
    cnt += remote;
  }
  atomicAdd(nremote, (unsigned long long)cnt);
}

__global__ void k_gather_scores(const double* __restrict__ scores, const std::uint32_t* __restrict__ order,
                                std::uint64_t cnt, double* __restrict__ out) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    out[i] = scores[order[i]];
}

__global__ void k_reorder_keys(const double* __restrict__ scores, const std::uint32_t* __restrict__ part_of,
                               std::uint64_t n, std::uint64_t* __restrict__ keys, std::uint32_t* __restrict__ ids) {
  for (std::uint64_t v = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (std::uint64_t)gridDim.x * blockDim.x) {
    keys[v] = desc_key(scores[(std::uint64_t)part_of[v] * n + v]);
    ids[v] = (std::uint32_t)v;
  }
}

__global__ void k_part_keys(const std::uint32_t* __restrict__ part_of, const std::uint32_t* __restrict__ ids,
                            std::uint64_t n, std::uint32_t* __restrict__ keys) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    keys[i] = part_of[ids[i]];
}

unsigned grid_for(std::uint64_t work, int device) {
  const std::uint64_t g = (work + 255) / 256;
  const std::uint64_t cap = (std::uint64_t)sm_count(device) * 16;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <class K, class V>
void radix_sort_pairs(DevBuf& k_in, DevBuf& k_out, DevBuf& v_in, DevBuf& v_out, std::uint64_t n, int end_bit,
                      cudaStream_t st) {
  std::size_t tmp = 0;
  VK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k_in.as<K>(), k_out.as<K>(), v_in.as<V>(),
                                          v_out.as<V>(), (std::int64_t)n, 0, end_bit, st));
  DevBuf t(tmp);
  VK_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, k_in.as<K>(), k_out.as<K>(), v_in.as<V>(), v_out.as<V>(),
                                          (std::int64_t)n, 0, end_bit, st));
  count_launch(4);
}

// ---- synthetic feature rows (identical to oracle vp_feature_*) ----
__device__ __forceinline__ std::uint64_t feat_bits(std::uint64_t seed, std::uint64_t v, std::uint32_t j,
                                                   std::uint32_t D) {
  return mix64(seed ^ mix64(v * (std::uint64_t)D + j));
}

__global__ void k_synth_rows(const std::uint32_t* __restrict__ ids, std::uint64_t rows, std::uint32_t D,
                             int fp16, std::uint64_t seed, void* __restrict__ out) {
  const std::uint64_t total = rows * D;
  for (std::uint64_t e = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t r = e / D;
    const std::uint32_t j = (std::uint32_t)(e - r * D);
    const std::uint64_t x = feat_bits(seed, ids[r], j, D);
    if (fp16)
      static_cast<__half*>(out)[e] = __float2half_rn((float)(x >> 53) * 0x1.0p-10f - 1.0f);
    else
      static_cast<float*>(out)[e] = (float)(x >> 40) * 0x1.0p-23f - 1.0f;
  }
}

// Cache row of v in partition k's store (after its n_local local rows), from
// the cache index: cache rows are stored in ascending vertex id, so the row
// is the word's first-member rank plus the members below v in the word. A
// gather tile covers a contiguous vertex range, so its index words (and the
// new_id entries every row reads) are shared by all the wave's minibatches
// and stay in L2 -- unlike a u32 slot map per partition, whose entries for a
// minibatch's rows are scattered sectors (C4: ~1.5 GB of DRAM reads a wave).
__device__ __forceinline__ bool cache_rank(const uint4* __restrict__ cw, std::uint32_t v, std::uint32_t& rank) {
  const uint4 c = __ldg(cw + (v >> 6));
  const unsigned long long bits = ((unsigned long long)c.y << 32) | c.x;
  const unsigned long long below = bits & ((1ull << (v & 63)) - 1ull);
  rank = c.z + (std::uint32_t)__popcll(below);
  return (bits >> (v & 63)) & 1ull;
}

// ---- classify + gather ----
constexpr std::uint32_t kGatherTileWords = 64;  // 4096 vertices per (tile, minibatch) CTA
struct GatherParams {
  const std::uint32_t* all;
  std::uint64_t all_stride;
  const std::uint32_t* all_count;
  const char* desc;          // WaveDesc array; partition at desc + mb*desc_stride
  std::uint64_t desc_stride;
  const char* const* base;   // [K] local-row base of each partition (local or peer)
  const uint4* const* cword;         // [K] cache index (resident partitions)
  const std::uint32_t* nlocal;       // [K]
  const std::uint32_t* part_of;
  const std::uint32_t* owner_row;
  const std::uint32_t* new_id;       // [n] rstart[part_of[v]] + owner_row[v]
  const std::uint32_t* rstart;       // [K+1]
  std::uint32_t K;
  const unsigned char* peer_mask;    // [K] 1 if the partition's rows live on another GPU
  const unsigned long long* const* rmask;  // [K] remote-miss masks (resident partitions)
  char* out;
  std::uint64_t out_stride_bytes;
  std::uint64_t row_bytes;
  std::uint32_t V;                   // vector elements per row
  std::uint32_t magic32;             // ceil(2^32 / V): row = umulhi(e, magic32) for e < 32*V
  unsigned long long* counts;        // [nmb][4]
  // vertex-tile schedule: CTA b serves minibatch b % nmb, vertex tile b / nmb
  const uint4* all_rank;             // [nmb][W] {bits, rank prefix} of all_vertices
  // sparse frontiers instead: rank of each all-level bucket's first vertex
  // [nmb][tb_nb + 1]; a gather tile is tb_group consecutive buckets
  const std::uint32_t* tile_base;
  std::uint32_t tb_nb, tb_group, tb_split;
  std::uint64_t W;
  std::uint32_t nmb, tiles, tile_words;
  // deduplicated remote rows: staged[rank of new_id[v] in the wave's remote
  // set] -- ranked in global row order so the pull streams each owner's
  // store in ascending address order
  const unsigned long long* ubits;
  const std::uint32_t* uprefix;
  const char* staging;
  std::uint32_t stage_cap;
};

// The all_vertices index range [lo, hi) of vertex tile `tile` of minibatch
// mb: from the dense rank words at tile starts, or (sparse frontiers) from the
// all-level bucket bases.
__device__ __forceinline__ void tile_range(const GatherParams& p, std::uint32_t mb, std::uint32_t tile,
                                           std::uint32_t cnt, std::uint32_t& lo, std::uint32_t& hi) {
  if (p.tile_base) {
    const std::uint32_t* tb = p.tile_base + (std::uint64_t)mb * (p.tb_nb + 1);
    if (p.tb_split > 1) {  // part tile % split of bucket tile / split, by rows
      const std::uint32_t b = tile / p.tb_split, part = tile % p.tb_split;
      const std::uint32_t l = tb[b], h = tb[b + 1];
      lo = l + (std::uint32_t)((std::uint64_t)(h - l) * part / p.tb_split);
      hi = l + (std::uint32_t)((std::uint64_t)(h - l) * (part + 1) / p.tb_split);
      return;
    }
    const std::uint32_t b0 = tile * p.tb_group;
    lo = b0 < p.tb_nb ? tb[b0] : cnt;
    hi = tb[min(b0 + p.tb_group, p.tb_nb)];
    return;
  }
  const uint4* rk = p.all_rank + mb * p.W;
  const std::uint64_t w0 = (std::uint64_t)tile * p.tile_words, w1 = w0 + p.tile_words;
  lo = w0 < p.W ? rk[w0].z : cnt;
  hi = w1 < p.W ? rk[w1].z : cnt;
}

constexpr std::uint32_t kMagicExactV = 11585;  // largest V with V*V < 2^27
constexpr unsigned kPullCtasPrefetch = 2;  // pull CTAs per SM beside a running gather

// Row of flattened element e (< 32 V) of a warp's 32 rows: umulhi with
// ceil(2^32/V) is exact while V*V < 2^27 (V <= 11585); above that it can
// overshoot by one, which the fix-up corrects.
__device__ __forceinline__ std::uint32_t row_of(std::uint32_t e, std::uint32_t V, std::uint32_t magic,
                                                std::uint32_t fix) {
  if (V == 1) return e;
  std::uint32_t row = __umulhi(e, magic);
  if (fix) row -= (row * V > e) ? 1u : 0u;
  return row;
}

// Owner partition of global row g: the last k with rstart[k] <= g (K+1
// range starts, staged in shared memory when K <= kSmemParts).
constexpr std::uint32_t kSmemParts = 256;
__device__ __forceinline__ std::uint32_t owner_of(const std::uint32_t* rs, std::uint32_t K, std::uint32_t g) {
  std::uint32_t lo = 0, hi = K;
  while (hi - lo > 1) {
    const std::uint32_t mid = (lo + hi) >> 1;
    if (rs[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ const std::uint32_t* stage_rstart(const GatherParams& p, std::uint32_t* sm) {
  if (p.K + 1 > kSmemParts) return p.rstart;
  for (std::uint32_t i = threadIdx.x; i <= p.K; i += blockDim.x) sm[i] = p.rstart[i];
  __syncthreads();
  return sm;
}

// Row copies move 16/4/2-byte vectors. Source rows are read through L1
// without allocating and with an L2 evict_last policy (a row read for one
// minibatch of the wave stays in L2 for the others; C3: 5.60 -> 5.23 ms);
// gathered rows are written evict-first so they do not evict the graph and
// cache index from L2. Measured no better, and removed: plain / L1::no_allocate
// stores, evict_normal loads, L2 hints on the index loads.
template <class T>
__device__ __forceinline__ T ld_row(const T* p, std::uint64_t pol) {
  if constexpr (sizeof(T) == 16) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
  } else {
    return __ldg(p);
  }
}
template <class T>
__device__ __forceinline__ void st_row(T* p, const T& v) {
  if constexpr (sizeof(T) == 16)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else
    __stcs(p, v);
}
// Plain coherent loads for rows that live on a peer GPU (read over NVLink
// through a CUDA IPC mapping): the non-coherent / cache-hinted path above
// measured ~40x slower there.
template <class T>
__device__ __forceinline__ T ld_peer(const T* p) {
  if constexpr (sizeof(T) == 16) {
    uint4 r;
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
  } else if constexpr (sizeof(T) == 4) {
    std::uint32_t r;
    asm volatile("ld.global.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
  } else {
    std::uint16_t r;
    asm volatile("ld.global.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
  }
}
// Source pointers of peer rows carry tag bit 0 (rows are >= 2-byte aligned).
template <class T>
__device__ __forceinline__ const T* tag_peer(const T* p) {
  return reinterpret_cast<const T*>(reinterpret_cast<std::uintptr_t>(p) | 1u);
}

__device__ __forceinline__ std::uint64_t evict_last_policy() {
  std::uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Flat copy of a warp's group of `rows` rows (V vectors each) from the 32
// source pointers in src[] to consecutive output rows: element e of the
// group is vector e % V of row e / V, kUnroll independent loads in flight
// per lane, fully coalesced stores. FIX: V > 11585 (see row_of).
template <class T, int kUnroll, bool FIX>
__device__ __forceinline__ void copy_group(const T* const* src, T* dst, std::uint32_t rows, std::uint32_t V,
                                           std::uint32_t magic, std::uint64_t pol) {
  const std::uint32_t total = rows * V;
  for (std::uint32_t e0 = threadIdx.x & 31; e0 < total; e0 += 32 * kUnroll) {
    T val[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const std::uint32_t e = e0 + 32 * u;
      if (e < total) {
        const std::uint32_t row = row_of(e, V, magic, FIX);
        const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(src[row]);
        const T* sp = reinterpret_cast<const T*>(a & ~std::uintptr_t(1)) + (e - row * V);
        val[u] = (a & 1u) ? ld_peer(sp) : ld_row(sp, pol);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const std::uint32_t e = e0 + 32 * u;
      if (e < total) st_row(dst + e, val[u]);
    }
  }
}

// One warp per group of 32 consecutive output rows: lanes first resolve the
// 32 source rows in parallel (classify: local row, cache row, or the
// owner partition's row, local HBM or a peer GPU over NVLink), then the warp
// copies the group as one flat, fully coalesced range of 32*V vectors with
// kUnroll independent loads in flight per lane.
// Multi-GPU miss exchange, step 1: the union of the wave's remote misses
// (rows whose owner partition lives on another GPU and that are neither
// local nor cached for the minibatch's partition) as a bitmap over vertices.
__global__ void __launch_bounds__(256) k_remote_mark(GatherParams p, unsigned long long* __restrict__ ubits) {
  __shared__ std::uint32_t s_rs[kSmemParts];
  const std::uint32_t* rs = stage_rstart(p, s_rs);
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t k = *reinterpret_cast<const std::uint32_t*>(p.desc + mb * p.desc_stride);
  const std::uint32_t cnt = p.all_count[mb];
  const std::uint32_t* all = p.all + mb * p.all_stride;
  const uint4* cw = p.cword[k];
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < cnt; r += gridDim.x * blockDim.x) {
    const std::uint32_t v = __ldg(all + r);
    const std::uint32_t g = __ldg(p.new_id + v);
    std::uint32_t cr;
    // owner on a peer GPU (so not k, which is resident) and not cached for k
    if (p.peer_mask[owner_of(rs, p.K, g)] && !cache_rank(cw, v, cr)) atomicOr(ubits + (g >> 6), 1ull << (g & 63));
  }
}

// Step 1 from the sampler's bitmaps (dense all-level rank words), in two
// passes: (a) per (vertex word, chunk of kMarkChunk minibatches) OR the
// all-vertex bits masked by each minibatch partition's remote-miss mask into
// a vertex-space union; (b) per union word, set each vertex's bit in global
// row order and clear the word for the next wave. Reads M*W*16 B of rank
// words instead of every row's id, new_id and cache word.
constexpr std::uint32_t kMarkChunk = 8;
__global__ void __launch_bounds__(256) k_remote_union(GatherParams p, unsigned long long* __restrict__ vbits) {
  const std::uint64_t w = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (w >= p.W) return;
  const std::uint32_t mb0 = blockIdx.y * kMarkChunk;
  unsigned long long u = 0;
#pragma unroll
  for (std::uint32_t i = 0; i < kMarkChunk; ++i) {
    const std::uint32_t mb = mb0 + i;
    if (mb < p.nmb) {
      const std::uint32_t k = *reinterpret_cast<const std::uint32_t*>(p.desc + mb * p.desc_stride);
      const uint4 r = __ldg(p.all_rank + mb * p.W + w);
      u |= (((unsigned long long)r.y << 32) | r.x) & __ldg(p.rmask[k] + w);
    }
  }
  if (u) atomicOr(vbits + w, u);
}
__global__ void __launch_bounds__(256) k_remote_to_rows(const GatherParams p, unsigned long long* __restrict__ vbits,
                                                        unsigned long long* __restrict__ ubits) {
  for (std::uint64_t w = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; w < p.W;
       w += (std::uint64_t)gridDim.x * blockDim.x) {
    unsigned long long u = vbits[w];
    if (!u) continue;
    vbits[w] = 0ull;
    while (u) {
      const int b = __ffsll(u) - 1;
      u &= u - 1;
      const std::uint32_t g = __ldg(p.new_id + (w * 64 + b));
      atomicOr(ubits + (g >> 6), 1ull << (g & 63));
    }
  }
}

__global__ void k_remote_miss_mask(const uint4* __restrict__ cword, const std::uint32_t* __restrict__ part_of,
                                   const unsigned char* __restrict__ peer_mask, std::uint64_t n,
                                   unsigned long long* __restrict__ out) {
  const std::uint64_t W = (n + 63) / 64;
  for (std::uint64_t w = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; w < W;
       w += (std::uint64_t)gridDim.x * blockDim.x) {
    const uint4 c = cword[w];
    const unsigned long long cached = ((unsigned long long)c.y << 32) | c.x;
    unsigned long long m = 0;
    for (int b = 0; b < 64; ++b) {
      const std::uint64_t v = w * 64 + b;
      // owner on a peer GPU (never the resident partition itself), not cached
      if (v < n && peer_mask[part_of[v]] && !((cached >> b) & 1ull)) m |= 1ull << b;
    }
    out[w] = m;
  }
}

__global__ void k_word_popc(const unsigned long long* __restrict__ bits, std::uint64_t W,
                            std::uint32_t* __restrict__ out) {
  for (std::uint64_t w = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; w < W;
       w += (std::uint64_t)gridDim.x * blockDim.x)
    out[w] = (std::uint32_t)__popcll(bits[w]);
}

__global__ void k_emit_list(const unsigned long long* __restrict__ bits, const std::uint32_t* __restrict__ prefix,
                            std::uint64_t W, std::uint32_t* __restrict__ list) {
  for (std::uint64_t w = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; w < W;
       w += (std::uint64_t)gridDim.x * blockDim.x) {
    unsigned long long x = bits[w];
    std::uint32_t pos = prefix[w];
    while (x) {
      const int b = __ffsll(x) - 1;
      x &= x - 1;
      list[pos++] = (std::uint32_t)(w * 64 + b);
    }
  }
}

// Step 2: one NVLink read per distinct remote row into the staging buffer
// (warp per 32 rows, 128-bit copies); the gather then serves every
// minibatch's remote misses from local HBM.
template <class T, int kUnroll, bool FIX>
__global__ void __launch_bounds__(256) k_remote_pull(GatherParams p, const std::uint32_t* __restrict__ list,
                                                     const std::uint32_t* __restrict__ count_ptr, T* __restrict__ staging) {
  __shared__ const T* s_src[8][32];
  __shared__ std::uint32_t s_rs[kSmemParts];
  const std::uint32_t* rs = stage_rstart(p, s_rs);
  const std::uint32_t cnt = min(*count_ptr, p.stage_cap);
  const std::uint64_t rowv = p.row_bytes / sizeof(T);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const std::uint64_t pol = evict_last_policy();
  const std::uint32_t gw = blockIdx.x * (blockDim.x >> 5) + w, nw = gridDim.x * (blockDim.x >> 5);
  for (std::uint32_t r0 = gw * 32; r0 < cnt; r0 += nw * 32) {
    const std::uint32_t r = r0 + lane;
    const T* src = nullptr;
    if (r < cnt) {
      const std::uint32_t g = __ldg(list + r);  // global row order
      const std::uint32_t o = owner_of(rs, p.K, g);
      src = tag_peer(reinterpret_cast<const T*>(p.base[o]) + (std::uint64_t)(g - rs[o]) * rowv);  // NVLink
    }
    s_src[w][lane] = src;
    __syncwarp();
    copy_group<T, kUnroll, FIX>(s_src[w], staging + (std::uint64_t)r0 * p.V, min(32u, cnt - r0), p.V, p.magic32, pol);
    __syncwarp();
  }
}

// STAGED false: every row is read where it lives -- local HBM, or a peer
// GPU's store over NVLink (CUDA IPC mapping) for remote misses; true: the
// remote misses of the wave were pulled into the staging buffer by the
// deduplicating miss exchange and are read from there.
template <class T, bool STAGED, bool FIX>
__global__ void __launch_bounds__(256, sizeof(T) == 16 ? 4 : 1) k_gather(GatherParams p) {
  constexpr int kUnroll = 8;
  __shared__ const T* s_src[8][32];
  __shared__ unsigned sh[4][8];
  __shared__ std::uint32_t s_rs[kSmemParts];
  const std::uint32_t* rs = stage_rstart(p, s_rs);
  const std::uint64_t pol = evict_last_policy();
  // Units are (vertex tile, minibatch) pairs, vertex-tile-major with the
  // minibatch fastest: the CTAs resident at any moment serve the same vertex
  // range for every minibatch of the wave, so a feature row needed by several
  // minibatches is read from HBM once and hit in L2 by the others
  // (all_vertices is sorted: a vertex range is a contiguous run of output rows).
  const std::uint32_t unit = blockIdx.x;
  const std::uint32_t mb = unit % p.nmb;
  const std::uint32_t tile = unit / p.nmb;
  const std::uint32_t k = *reinterpret_cast<const std::uint32_t*>(p.desc + mb * p.desc_stride);
  const std::uint32_t cnt = p.all_count[mb];
  std::uint32_t lo, hi;
  tile_range(p, mb, tile, cnt, lo, hi);
  const std::uint32_t* all = p.all + mb * p.all_stride;
  const uint4* cw = p.cword[k];
  const std::uint32_t nl = p.nlocal[k], rk = rs[k];
  const T* store = reinterpret_cast<const T*>(p.base[k]);
  T* out = reinterpret_cast<T*>(p.out + mb * p.out_stride_bytes);
  const std::uint64_t rowv = p.row_bytes / sizeof(T);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned c_local = 0, c_cache = 0, c_miss = 0, c_peer = 0;
  for (std::uint32_t r0 = lo + w * 32; r0 < hi; r0 += (blockDim.x >> 5) * 32) {
    const std::uint32_t r = r0 + lane;
    const T* src = nullptr;
    if (r < hi) {
      // classify (commsim.cpp:61-73): the owner of global row g = new_id[v]
      // is k -> local row; else cached for k -> cache row; else the owner's
      // row in global row order
      const std::uint32_t v = __ldg(all + r);
      const std::uint32_t g = __ldg(p.new_id + v);
      const std::uint32_t o = owner_of(rs, p.K, g);
      std::uint32_t cr;
      if (o == k) {
        src = store + (std::uint64_t)(g - rk) * rowv;
        ++c_local;
      } else if (cache_rank(cw, v, cr)) {
        src = store + (std::uint64_t)(nl + cr) * rowv;
        ++c_cache;
      } else {
        src = reinterpret_cast<const T*>(p.base[o]) + (std::uint64_t)(g - rs[o]) * rowv;
        ++c_miss;
        if (p.peer_mask[o]) {  // owned by a partition on another GPU
          ++c_peer;
          src = tag_peer(src);  // read over NVLink unless staged below
        }
        if (STAGED && p.peer_mask[o]) {  // pulled once per wave into local staging
          const std::uint32_t wq = g >> 6;
          const std::uint32_t idx = __ldg(p.uprefix + wq) +
                                    (std::uint32_t)__popcll(__ldg(p.ubits + wq) & ((1ull << (g & 63)) - 1ull));
          if (idx < p.stage_cap)  // else past the staging capacity: the direct NVLink read above
            src = reinterpret_cast<const T*>(p.staging) + (std::uint64_t)idx * rowv;
        }
      }
    }
    s_src[w][lane] = src;
    __syncwarp();
    copy_group<T, kUnroll, FIX>(s_src[w], out + (std::uint64_t)r0 * p.V, min(32u, hi - r0), p.V, p.magic32, pol);
    __syncwarp();
  }
  // block-reduce the class counts, one atomic per class per CTA
  unsigned vals[4] = {c_local, c_cache, c_miss, c_peer};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned x = __reduce_add_sync(0xffffffffu, vals[q]);
    if ((threadIdx.x & 31) == 0) sh[q][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
    if (t) atomicAdd(p.counts + mb * 4 + threadIdx.x, t);
  }
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" {

int vk_rank_by_scores(int device, uint64_t n, const uint32_t* part_of, uint32_t k, const double* scores,
                      uint64_t n_scores, uint32_t* order_out, double* score_out, uint64_t* count_out) {
  return guard([&] {
    if (!part_of || !scores || !order_out || !count_out) raise(VK_ERR_PARAMETER, "null argument");
    if (n_scores != n) raise(VK_ERR_SHAPE, "score vector length does not match vertex count");  // policies.cpp:135-136
    DeviceGuard dg(device);
    cudaStream_t st;
    VK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      DevBuf dsc(n * 8), dpart(n * 4), k0(n * 8), k1(n * 8), i0(n * 4), i1(n * 4), cnt(8);
      VK_CUDA(cudaMemcpyAsync(dsc.p, scores, n * 8, cudaMemcpyHostToDevice, st));
      VK_CUDA(cudaMemcpyAsync(dpart.p, part_of, n * 4, cudaMemcpyHostToDevice, st));
      VK_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
      k_rank_keys<<<grid_for(n, device), 256, 0, st>>>(dsc.as<double>(), dpart.as<std::uint32_t>(), n, k,
                                                       k0.as<std::uint64_t>(), i0.as<std::uint32_t>(),
                                                       cnt.as<unsigned long long>());
      count_launch();
      VK_LAUNCH_CHECK();
      radix_sort_pairs<std::uint64_t, std::uint32_t>(k0, k1, i0, i1, n, 64, st);
      unsigned long long c = 0;
      VK_CUDA(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
      VK_CUDA(cudaStreamSynchronize(st));
      if (c) {
        VK_CUDA(cudaMemcpyAsync(order_out, i1.p, c * 4, cudaMemcpyDeviceToHost, st));
        if (score_out) {
          k_gather_scores<<<grid_for(c, device), 256, 0, st>>>(dsc.as<double>(), i1.as<std::uint32_t>(), c,
                                                               k0.as<double>());
          count_launch();
          VK_LAUNCH_CHECK();
          VK_CUDA(cudaMemcpyAsync(score_out, k0.p, c * 8, cudaMemcpyDeviceToHost, st));
        }
      }
      VK_CUDA(cudaStreamSynchronize(st));
      *count_out = c;
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
  });
}

int vk_build_reorder(int device, uint64_t n, uint32_t K, const uint32_t* part_of, const double* scores,
                     uint32_t* old_of_new, uint64_t* ranges) {
  return guard([&] {
    if (!part_of || !scores || !old_of_new || !ranges) raise(VK_ERR_PARAMETER, "null argument");
    if (K == 0) raise(VK_ERR_PARAMETER, "partition count must be >= 1");
    std::vector<std::uint64_t> cnt(K, 0);
    for (std::uint64_t v = 0; v < n; ++v) {
      if (part_of[v] >= K) raise(VK_ERR_FORMAT, "partition label out of range");
      cnt[part_of[v]]++;
    }
    DeviceGuard dg(device);
    cudaStream_t st;
    VK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      DevBuf dsc(n * 8 * K), dpart(n * 4), k0(n * 8), k1(n * 8), i0(n * 4), i1(n * 4), p0(n * 4), p1(n * 4);
      VK_CUDA(cudaMemcpyAsync(dsc.p, scores, n * 8 * K, cudaMemcpyHostToDevice, st));
      VK_CUDA(cudaMemcpyAsync(dpart.p, part_of, n * 4, cudaMemcpyHostToDevice, st));
      k_reorder_keys<<<grid_for(n, device), 256, 0, st>>>(dsc.as<double>(), dpart.as<std::uint32_t>(), n,
                                                          k0.as<std::uint64_t>(), i0.as<std::uint32_t>());
      count_launch();
      VK_LAUNCH_CHECK();
      radix_sort_pairs<std::uint64_t, std::uint32_t>(k0, k1, i0, i1, n, 64, st);
      k_part_keys<<<grid_for(n, device), 256, 0, st>>>(dpart.as<std::uint32_t>(), i1.as<std::uint32_t>(), n,
                                                       p0.as<std::uint32_t>());
      count_launch();
      VK_LAUNCH_CHECK();
      int bits = 1;
      while ((1ull << bits) < K) ++bits;
      radix_sort_pairs<std::uint32_t, std::uint32_t>(p0, p1, i1, i0, n, bits, st);
      VK_CUDA(cudaMemcpyAsync(old_of_new, i0.p, n * 4, cudaMemcpyDeviceToHost, st));
      VK_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
    std::uint64_t pos = 0;
    for (std::uint32_t k = 0; k < K; ++k) {
      ranges[2 * k] = pos;
      pos += cnt[k];
      ranges[2 * k + 1] = pos;
    }
  });
}

int vk_plane_create(int device, uint64_t n, uint32_t K, uint32_t dim, int dtype, const uint32_t* part_of,
                    const uint32_t* old_of_new, const uint64_t* ranges, vk_plane* out) {
  return guard([&] {
    if (!part_of || !old_of_new || !ranges || !out) raise(VK_ERR_PARAMETER, "null argument");
    if (K == 0 || dim == 0 || n == 0) raise(VK_ERR_PARAMETER, "n, K and dim must be >= 1");
    if (dtype != VK_F32 && dtype != VK_F16) raise(VK_ERR_PARAMETER, "dtype must be VK_F32 or VK_F16");
    // owner_row[v] = position of v inside its partition's range (reorder map)
    std::vector<std::uint32_t> owner(n, VK_MISS);
    std::vector<std::uint64_t> rs(K), re(K);
    std::uint64_t prev = 0;
    for (std::uint32_t k = 0; k < K; ++k) {
      rs[k] = ranges[2 * k];
      re[k] = ranges[2 * k + 1];
      if (rs[k] != prev || re[k] < rs[k] || re[k] > n) raise(VK_ERR_SHAPE, "reorder ranges malformed");
      prev = re[k];
      for (std::uint64_t i = rs[k]; i < re[k]; ++i) {
        const std::uint32_t v = old_of_new[i];
        if (v >= n || owner[v] != VK_MISS) raise(VK_ERR_SHAPE, "old_of_new is not a permutation");
        if (part_of[v] != k) raise(VK_ERR_SHAPE, "reorder range does not match partition labels");
        owner[v] = (std::uint32_t)(i - rs[k]);
      }
    }
    if (prev != n) raise(VK_ERR_SHAPE, "reorder map size does not match vertex count");
    DeviceGuard dg(device);
    auto* p = new vk_plane_s();
    try {
      p->device = device;
      p->n = n;
      p->K = K;
      p->dim = dim;
      p->dtype = dtype;
      p->row_bytes = (std::uint64_t)dim * (dtype == VK_F16 ? 2 : 4);
      p->rstart = rs;
      p->rend = re;
      p->old_of_new.assign(old_of_new, old_of_new + n);
      p->parts.resize(K);
      VK_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
      {
        // the aux stream (miss exchange) runs at the highest priority: its
        // CTAs take SM slots as soon as the running gather's retire, so a
        // prefetched exchange overlaps the HBM-bound gather instead of
        // waiting for it to drain
        int lo = 0, hi = 0;
        VK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VK_CUDA(cudaStreamCreateWithPriority(&p->aux, cudaStreamNonBlocking, hi));
        VK_CUDA(cudaEventCreateWithFlags(&p->after_ev, cudaEventDisableTiming));
      }
      p->part_of.alloc(n * 4);
      p->owner_row.alloc(n * 4);
      p->new_id.alloc(n * 4);
      p->d_rstart.alloc((K + 1) * 4);
      std::vector<std::uint32_t> nid(n), rst(K + 1);
      for (std::uint32_t k = 0; k < K; ++k) rst[k] = (std::uint32_t)rs[k];
      rst[K] = (std::uint32_t)n;
      for (std::uint64_t i = 0; i < n; ++i) nid[old_of_new[i]] = (std::uint32_t)i;
      VK_CUDA(cudaMemcpyAsync(p->part_of.p, part_of, n * 4, cudaMemcpyHostToDevice, p->stream));
      VK_CUDA(cudaMemcpyAsync(p->owner_row.p, owner.data(), n * 4, cudaMemcpyHostToDevice, p->stream));
      VK_CUDA(cudaMemcpyAsync(p->new_id.p, nid.data(), n * 4, cudaMemcpyHostToDevice, p->stream));
      VK_CUDA(cudaMemcpyAsync(p->d_rstart.p, rst.data(), (K + 1) * 4, cudaMemcpyHostToDevice, p->stream));
      p->d_base.alloc(K * sizeof(void*));
      p->d_cword.alloc(K * sizeof(void*));
      p->d_nlocal.alloc(K * 4 + K);  // u32 nlocal[K] then u8 peer_mask[K]
      VK_CUDA(cudaMemsetAsync(p->d_base.p, 0, p->d_base.bytes, p->stream));
      VK_CUDA(cudaMemsetAsync(p->d_cword.p, 0, p->d_cword.bytes, p->stream));
      VK_CUDA(cudaMemsetAsync(p->d_nlocal.p, 0, p->d_nlocal.bytes, p->stream));
      VK_CUDA(cudaStreamSynchronize(p->stream));
    } catch (...) {
      vk_plane_destroy(p);
      throw;
    }
    *out = p;
  });
}

int vk_plane_destroy(vk_plane p) {
  return guard([&] {
    if (!p) return;
    DeviceGuard dg(p->device);
    // gathers on caller streams and prefetched exchanges may still read peer
    // memory: drain the device before the IPC mappings go away
    cudaDeviceSynchronize();
    for (auto& part : p->parts)
      if (part.peer) cudaIpcCloseMemHandle(part.peer);
    if (p->stream) cudaStreamDestroy(p->stream);
    if (p->aux) cudaStreamDestroy(p->aux);
    if (p->after_ev) cudaEventDestroy(p->after_ev);
    delete p;
  });
}

namespace {

void publish_tables(vk_plane_s& p) {
  std::vector<const void*> base(p.K, nullptr), cword(p.K, nullptr);
  std::vector<unsigned char> nl(p.K * 4 + p.K, 0);
  for (std::uint32_t k = 0; k < p.K; ++k) {
    const auto& q = p.parts[k];
    if (q.resident) {
      base[k] = q.store.p;
      cword[k] = q.cword.p;
      const std::uint32_t x = (std::uint32_t)q.n_local;
      std::memcpy(nl.data() + 4 * k, &x, 4);
    } else if (q.attached) {
      base[k] = q.peer;
      nl[p.K * 4 + k] = 1;
    }
  }
  VK_CUDA(cudaMemcpyAsync(p.d_base.p, base.data(), p.K * sizeof(void*), cudaMemcpyHostToDevice, p.stream));
  VK_CUDA(cudaMemcpyAsync(p.d_cword.p, cword.data(), p.K * sizeof(void*), cudaMemcpyHostToDevice, p.stream));
  VK_CUDA(cudaMemcpyAsync(p.d_nlocal.p, nl.data(), nl.size(), cudaMemcpyHostToDevice, p.stream));
  std::vector<const void*> rm(p.K, nullptr);
  const std::uint64_t W = (p.n + 63) / 64;
  for (std::uint32_t k = 0; k < p.K; ++k) {
    auto& q = p.parts[k];
    if (!q.resident) continue;
    if (!q.rmask.p) q.rmask.alloc(W * 8);
    k_remote_miss_mask<<<grid_for(W, p.device), 256, 0, p.stream>>>(
        q.cword.as<uint4>(), p.part_of.as<std::uint32_t>(), p.d_nlocal.as<unsigned char>() + 4 * p.K, p.n,
        q.rmask.as<unsigned long long>());
    VK_LAUNCH_CHECK();
    rm[k] = q.rmask.p;
  }
  if (!p.d_rmask.p) p.d_rmask.alloc(p.K * sizeof(void*));
  VK_CUDA(cudaMemcpyAsync(p.d_rmask.p, rm.data(), p.K * sizeof(void*), cudaMemcpyHostToDevice, p.stream));
  VK_CUDA(cudaStreamSynchronize(p.stream));
}

}  // namespace

int vk_plane_load_partition(vk_plane p, uint32_t k, const uint32_t* cache_ids, uint64_t n_cache,
                            const void* features, uint64_t feature_seed) {
  return guard([&] {
    if (!p) raise(VK_ERR_PARAMETER, "null plane");
    if (k >= p->K) raise(VK_ERR_CONFIG, "partition index out of range");
    if (n_cache && !cache_ids) raise(VK_ERR_PARAMETER, "null cache ids");
    auto& q = p->parts[k];
    const std::uint64_t n = p->n;
    const std::uint64_t nl = p->rend[k] - p->rstart[k];
    // cache ids: remote, distinct, in range (a ranking prefix always is)
    std::vector<std::uint64_t> bits((n + 63) / 64, 0);
    std::vector<std::uint32_t> part_host(n);
    DeviceGuard dg(p->device);
    VK_CUDA(cudaMemcpy(part_host.data(), p->part_of.p, n * 4, cudaMemcpyDeviceToHost));
    for (std::uint64_t i = 0; i < n_cache; ++i) {
      const std::uint32_t v = cache_ids[i];
      if (v >= n) raise(VK_ERR_FORMAT, "cached vertex id out of range");  // policies.cpp:191
      if (part_host[v] == k) raise(VK_ERR_PARAMETER, "cache holds a vertex local to its partition");
      if ((bits[v >> 6] >> (v & 63)) & 1u) raise(VK_ERR_PARAMETER, "duplicate cached vertex");
      bits[v >> 6] |= 1ull << (v & 63);
    }
    const std::uint64_t rows = nl + n_cache;
    if (rows >= VK_MISS) raise(VK_ERR_UNSUPPORTED, "too many rows in one partition store");
    // store rows: local rows in global row order, then the cached vertices
    // in ascending id (the cache index below ranks them by word)
    std::vector<std::uint32_t> ids(rows);
    std::memcpy(ids.data(), p->old_of_new.data() + p->rstart[k], nl * 4);
    {
      std::uint64_t r = nl;
      for (std::uint64_t w = 0; w < bits.size(); ++w)
        for (std::uint64_t x = bits[w]; x; x &= x - 1) ids[r++] = (std::uint32_t)(w * 64 + __builtin_ctzll(x));
    }
    const std::uint64_t W = bits.size();
    std::vector<std::uint32_t> cw(W * 4, 0u);
    std::uint32_t crank = 0;
    for (std::uint64_t w = 0; w < W; ++w) {
      cw[4 * w] = (std::uint32_t)bits[w];
      cw[4 * w + 1] = (std::uint32_t)(bits[w] >> 32);
      cw[4 * w + 2] = crank;
      crank += (std::uint32_t)__builtin_popcountll(bits[w]);
    }
    q.store.alloc(std::max<std::uint64_t>(rows, 1) * p->row_bytes);
    q.cword.alloc(std::max<std::uint64_t>(W, 1) * 16);
    DevBuf dids(std::max<std::uint64_t>(rows, 1) * 4);
    cudaStream_t st = p->stream;
    VK_CUDA(cudaMemcpyAsync(dids.p, ids.data(), rows * 4, cudaMemcpyHostToDevice, st));
    VK_CUDA(cudaMemcpyAsync(q.cword.p, cw.data(), W * 16, cudaMemcpyHostToDevice, st));
    if (features) {
      // stage the selected rows on the host, one H2D copy
      std::vector<unsigned char> rowsbuf(rows * p->row_bytes);
      const unsigned char* src = static_cast<const unsigned char*>(features);
      for (std::uint64_t r = 0; r < rows; ++r)
        std::memcpy(rowsbuf.data() + r * p->row_bytes, src + (std::uint64_t)ids[r] * p->row_bytes, p->row_bytes);
      VK_CUDA(cudaMemcpyAsync(q.store.p, rowsbuf.data(), rowsbuf.size(), cudaMemcpyHostToDevice, st));
      VK_CUDA(cudaStreamSynchronize(st));
    } else if (rows) {
      k_synth_rows<<<grid_for(rows * p->dim, p->device), 256, 0, st>>>(dids.as<std::uint32_t>(), rows, p->dim,
                                                                      p->dtype == VK_F16, feature_seed, q.store.p);
      count_launch();
      VK_LAUNCH_CHECK();
    }
    VK_CUDA(cudaStreamSynchronize(st));
    q.resident = true;
    q.attached = false;
    q.n_local = nl;
    q.n_cache = n_cache;
    q.cache_bits = std::move(bits);
    publish_tables(*p);
  });
}

int vk_plane_is_cached(vk_plane p, uint32_t k, uint32_t v, int* out) {
  return guard([&] {
    if (!p || !out) raise(VK_ERR_PARAMETER, "null argument");
    if (k >= p->K || !p->parts[k].resident) raise(VK_ERR_CONFIG, "partition not resident on this plane");
    if (v >= p->n) raise(VK_ERR_RANGE, "vertex id out of range");
    *out = (int)((p->parts[k].cache_bits[v >> 6] >> (v & 63)) & 1u);  // policies.hpp:58-60
  });
}

int vk_plane_export(vk_plane p, uint32_t k, void* handle64, uint64_t* rows) {
  return guard([&] {
    if (!p || !handle64) raise(VK_ERR_PARAMETER, "null argument");
    if (k >= p->K || !p->parts[k].resident) raise(VK_ERR_CONFIG, "partition not resident on this plane");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t h;
    VK_CUDA(cudaIpcGetMemHandle(&h, p->parts[k].store.p));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
    if (rows) *rows = p->parts[k].n_local;
  });
}

int vk_plane_attach(vk_plane p, uint32_t k, const void* handle64, uint64_t rows) {
  return guard([&] {
    if (!p || !handle64) raise(VK_ERR_PARAMETER, "null argument");
    if (k >= p->K) raise(VK_ERR_CONFIG, "partition index out of range");
    if (p->parts[k].resident) raise(VK_ERR_CONFIG, "partition already resident on this plane");
    if (rows != p->rend[k] - p->rstart[k]) raise(VK_ERR_SHAPE, "peer partition row count mismatch");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    void* ptr = nullptr;
    VK_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    auto& q = p->parts[k];
    if (q.peer) cudaIpcCloseMemHandle(q.peer);
    q.peer = ptr;
    q.attached = true;
    publish_tables(*p);
  });
}

int vk_plane_pulled_rows(vk_plane p, uint64_t* rows) {
  return guard([&] {
    if (!p || !rows) raise(VK_ERR_PARAMETER, "null argument");
    *rows = 0;
    if (!p->last_set) return;
    DeviceGuard dg(p->device);
    std::uint32_t c = 0;
    VK_CUDA(cudaDeviceSynchronize());
    VK_CUDA(cudaMemcpy(&c, p->last_set->uprefix.as<std::uint32_t>() + (p->n + 63) / 64, 4, cudaMemcpyDeviceToHost));
    *rows = c;
  });
}

int vk_plane_row_bytes(vk_plane p, uint64_t* row_bytes) {
  return guard([&] {
    if (!p || !row_bytes) raise(VK_ERR_PARAMETER, "null argument");
    *row_bytes = p->row_bytes;
  });
}

}  // extern "C"

namespace {

// The classify + gather of a sampler's last wave (prefetch_only = false), or
// only its multi-GPU miss exchange, issued on the plane's aux stream so it
// overlaps whatever the caller queues next (prefetch_only = true; a later
// gather of the same run then waits for it instead of exchanging again).
void gather_impl(vk_plane p, vk_sampler s, void* out_dev, uint64_t out_stride_rows, uint64_t* counts_dev,
                 vk_stream_t stream, bool prefetch_only) {
  {
    if (!p || !s || (!prefetch_only && (!out_dev || !counts_dev))) raise(VK_ERR_PARAMETER, "null argument");
    GatherParams gp{};
    std::uint32_t nmb = 0;
    vk_graph_s* g = nullptr;
    cudaStream_t last = nullptr;
    const std::uint32_t* parts = nullptr;
    sampler_internal(s, &gp.all, &gp.all_stride, &gp.all_count, &nmb, &parts, &g, &last);
    if (nmb == 0) raise(VK_ERR_PARAMETER, "sampler has not run");
    if (g->device != p->device) raise(VK_ERR_CONFIG, "sampler and plane live on different devices");
    if (g->n != p->n) raise(VK_ERR_SHAPE, "sampler graph and plane vertex counts differ");
    std::vector<std::uint32_t> hp;
    sampler_host_partitions(s, hp);
    for (std::uint32_t k : hp) {
      if (k >= p->K || !p->parts[k].resident)
        raise(VK_ERR_CONFIG, "minibatch partition " + std::to_string(k) + " is not resident on this plane");
    }
    for (std::uint32_t k = 0; k < p->K; ++k)
      if (!p->parts[k].resident && !p->parts[k].attached)
        raise(VK_ERR_CONFIG, "partition " + std::to_string(k) + " is neither resident nor attached");
    DeviceGuard dg(p->device);
    cudaStream_t st = prefetch_only ? p->aux
                                    : (stream ? static_cast<cudaStream_t>(stream) : (last ? last : p->stream));
    if (st != last) VK_CUDA(cudaStreamWaitEvent(st, sampler_done_event(s), 0));
    if (!prefetch_only) VK_CUDA(cudaMemsetAsync(counts_dev, 0, (std::uint64_t)nmb * 4 * 8, st));
    gp.desc = reinterpret_cast<const char*>(parts);
    gp.desc_stride = sampler_desc_stride();
    gp.base = reinterpret_cast<const char* const*>(p->d_base.p);
    gp.cword = reinterpret_cast<const uint4* const*>(p->d_cword.p);
    gp.nlocal = p->d_nlocal.as<std::uint32_t>();
    gp.peer_mask = p->d_nlocal.as<unsigned char>() + 4 * p->K;
    gp.part_of = p->part_of.as<std::uint32_t>();
    gp.owner_row = p->owner_row.as<std::uint32_t>();
    gp.new_id = p->new_id.as<std::uint32_t>();
    gp.rstart = p->d_rstart.as<std::uint32_t>();
    gp.K = p->K;
    gp.out = static_cast<char*>(out_dev);
    gp.out_stride_bytes = out_stride_rows * p->row_bytes;
    gp.row_bytes = p->row_bytes;
    gp.counts = reinterpret_cast<unsigned long long*>(counts_dev);
    const bool v16 = (p->row_bytes % 16 == 0) && ((std::uintptr_t)out_dev % 16 == 0);
    const bool v4 = (p->row_bytes % 4 == 0) && ((std::uintptr_t)out_dev % 4 == 0);
    // staged rows are plain rows of row_bytes in cudaMalloc'd memory: the
    // pull's vector width depends on the row size only
    const bool pv16 = p->row_bytes % 16 == 0, pv4 = p->row_bytes % 4 == 0;
    const std::uint64_t esz = v16 ? 16 : (v4 ? 4 : 2);
    gp.V = (std::uint32_t)(p->row_bytes / esz);
    if (gp.V >= (1u << 15)) raise(VK_ERR_UNSUPPORTED, "feature rows above 512 KiB are not supported");
    gp.magic32 = gp.V == 1 ? 0u : (std::uint32_t)((0xffffffffull / gp.V) + 1);  // ceil(2^32 / V)
    sampler_all_rank(s, &gp.all_rank, &gp.W);
    gp.rmask = p->d_rmask.as<const unsigned long long* const>();
    gp.nmb = nmb;
    // Gather tiles: a few thousand output rows per (tile, minibatch) unit.
    // Dense rank words exist at multiples of 64 words; the capacity
    // over-estimates the density (~1.8x at C3), so sparse neighbourhoods take
    // proportionally wider tiles (C3: 4096-vertex tiles 5.35 ms, 16384 5.08
    // ms), at most 2048 words: papers-scale waves have little row reuse
    // across minibatches. Sparse frontiers: whole all-level buckets.
    constexpr double kUnitRows = 3584.0;
    const double density = std::max(1e-9, (double)gp.all_stride / (double)p->n);
    const std::uint64_t want_words = std::min<std::uint64_t>(2048, (std::uint64_t)(kUnitRows / (64.0 * density)));
    const std::uint64_t tw = std::max<std::uint64_t>(kGatherTileWords, (want_words + 63) / 64 * 64);
    gp.tile_words = (std::uint32_t)tw;
    gp.tiles = (std::uint32_t)((gp.W + tw - 1) / tw);
    {
      std::uint32_t bbits = 0, nb = 0;
      gp.tile_base = sampler_tile_base(s, &bbits, &nb);
      if (gp.tile_base) {
        // papers-scale neighbourhoods have little row reuse across the
        // minibatches of a wave: ~1K-row units (C4: 2.2K-row buckets split in
        // two, 4.58 ms vs 4.93 ms for 4.4K-row units of two buckets)
        constexpr double kSparseUnitRows = 1024.0;
        const double rows_per_bucket = std::max(1.0, (double)gp.all_stride / (double)nb);
        gp.tb_nb = nb;
        if (rows_per_bucket > kSparseUnitRows) {
          gp.tb_group = 1;
          gp.tb_split = (std::uint32_t)std::min(64.0, std::round(rows_per_bucket / kSparseUnitRows));
          gp.tiles = nb * gp.tb_split;
        } else {
          gp.tb_group = (std::uint32_t)std::max(1.0, std::round(kSparseUnitRows / rows_per_bucket));
          gp.tb_split = 1;
          gp.tiles = (nb + gp.tb_group - 1) / gp.tb_group;
        }
      }
    }
    const std::uint64_t units = (std::uint64_t)gp.tiles * nmb;
    if (units >= (1ull << 31)) raise(VK_ERR_UNSUPPORTED, "too many gather tiles");
    bool staged = false;
    for (const auto& q : p->parts) staged |= q.attached;
    // With peers, the wave's remote misses are always exchanged (deduplicated,
    // pulled in ascending owner-row order) before the gather: even where the
    // dedup gains little (C4 at N=2: 11.0 M requests, 9.9 M distinct rows),
    // reading remote rows in random order straight from the gather measured
    // ~40x slower (199 ms per C4 wave) than the sorted pull.
    if (prefetch_only && !staged) return;  // nothing to exchange
    auto& ss = p->stage_sets[static_cast<const void*>(s)];
    const std::uint64_t run = sampler_run_id(s);
    const bool have_prefetch = staged && !prefetch_only && ss.prefetched == run;
    if (have_prefetch) {
      VK_CUDA(cudaStreamWaitEvent(st, ss.ready, 0));
      ss.prefetched = ~0ull;
      p->last_set = &ss;
      gp.ubits = ss.ubits.as<unsigned long long>();
      gp.uprefix = ss.uprefix.as<std::uint32_t>();
      gp.staging = ss.staging.as<char>();
      gp.stage_cap = (std::uint32_t)ss.stage_cap;
    }
    if (staged && !have_prefetch) {
      // miss exchange: union of the wave's remote misses -> distinct list ->
      // one NVLink pull per distinct row into local staging -> the gather
      // reads staged rows from HBM
      const std::uint64_t W = gp.W, n = p->n;
      auto ensure = [](DevBuf& b, std::size_t bytes) {
        if (b.bytes < bytes) b.alloc(bytes);
      };
      p->last_set = &ss;
      // a superseded prefetch of this stage set may still be running on aux
      if (ss.ready && st != p->aux) VK_CUDA(cudaStreamWaitEvent(st, ss.ready, 0));
      ss.prefetched = ~0ull;
      ensure(ss.ubits, W * 8);
      ensure(ss.uprefix, (W + 1) * 4);
      ensure(ss.ulist, n * 4);
      // staging holds at most half a wave's row capacity (bounded by the rows
      // owned by peers); distinct remote rows ranked past it are read from the
      // owner over NVLink by the gather itself
      {
        std::uint64_t remote_rows = 0;
        for (std::uint32_t k = 0; k < p->K; ++k)
          if (p->parts[k].attached) remote_rows += p->rend[k] - p->rstart[k];
        const std::uint64_t want = std::max<std::uint64_t>(1, std::min<std::uint64_t>(
            remote_rows, std::max<std::uint64_t>(1ull << 20, (std::uint64_t)nmb * gp.all_stride / 2)));
        if (ss.stage_cap < want) {
          ss.staging.alloc(want * p->row_bytes);
          ss.stage_cap = want;
        }
      }
      VK_CUDA(cudaMemsetAsync(ss.ubits.p, 0, W * 8, st));
      VK_CUDA(cudaMemsetAsync(ss.uprefix.as<std::uint32_t>() + W, 0, 4, st));
      if (sampler_all_rank_dense(s)) {
        // word-parallel marking from the dense all-level rank words
        if (!ss.vbits.p) {
          ss.vbits.alloc(W * 8);
          VK_CUDA(cudaMemsetAsync(ss.vbits.p, 0, W * 8, st));
        }
        k_remote_union<<<dim3((unsigned)ceil_div(W, 256), (unsigned)ceil_div(nmb, kMarkChunk)), 256, 0, st>>>(
            gp, ss.vbits.as<unsigned long long>());
        k_remote_to_rows<<<grid_for(W, p->device), 256, 0, st>>>(gp, ss.vbits.as<unsigned long long>(),
                                                                ss.ubits.as<unsigned long long>());
        count_launch(2);
      } else {
        const unsigned gx = (unsigned)std::max<std::uint64_t>(
            1, std::min<std::uint64_t>(ceil_div(gp.all_stride, 256), (std::uint64_t)sm_count(p->device) * 8 / nmb + 1));
        k_remote_mark<<<dim3(gx, nmb), 256, 0, st>>>(gp, ss.ubits.as<unsigned long long>());
        count_launch();
      }
      k_word_popc<<<grid_for(W, p->device), 256, 0, st>>>(ss.ubits.as<unsigned long long>(), W,
                                                          ss.uprefix.as<std::uint32_t>());
      exclusive_scan_u32(ss.uprefix.as<std::uint32_t>(), W + 1, ss.scan_tmp, st);
      k_emit_list<<<grid_for(W, p->device), 256, 0, st>>>(ss.ubits.as<unsigned long long>(),
                                                          ss.uprefix.as<std::uint32_t>(), W,
                                                          ss.ulist.as<std::uint32_t>());
      // NVLink-bound: a prefetched exchange shares the SMs with a running
      // gather (2 CTAs/SM, on the high-priority aux stream); inline, 8 CTAs/SM
      const unsigned pg = (unsigned)sm_count(p->device) * (prefetch_only ? kPullCtasPrefetch : 8);
      GatherParams pp = gp;  // staged rows are plain rows: the pull's vector width follows the row size
      auto pull = [&](auto tag, std::uint32_t esz) {
        using T = decltype(tag);
        pp.V = (std::uint32_t)(p->row_bytes / esz);
        pp.magic32 = pp.V == 1 ? 0u : (std::uint32_t)((0xffffffffull / pp.V) + 1);
        pp.stage_cap = (std::uint32_t)ss.stage_cap;
        if (pp.V > kMagicExactV)
          k_remote_pull<T, 8, true><<<pg, 256, 0, st>>>(pp, ss.ulist.as<std::uint32_t>(),
                                                        ss.uprefix.as<std::uint32_t>() + W, ss.staging.as<T>());
        else
          k_remote_pull<T, 8, false><<<pg, 256, 0, st>>>(pp, ss.ulist.as<std::uint32_t>(),
                                                         ss.uprefix.as<std::uint32_t>() + W, ss.staging.as<T>());
      };
      if (p->row_bytes % 16 == 0)
        pull(uint4{}, 16);
      else if (p->row_bytes % 4 == 0)
        pull(std::uint32_t{}, 4);
      else
        pull(std::uint16_t{}, 2);
      count_launch(3);
      VK_LAUNCH_CHECK();
      gp.ubits = ss.ubits.as<unsigned long long>();
      gp.uprefix = ss.uprefix.as<std::uint32_t>();
      gp.staging = ss.staging.as<char>();
      gp.stage_cap = (std::uint32_t)ss.stage_cap;
      if (prefetch_only) {
        if (!ss.ready) VK_CUDA(cudaEventCreateWithFlags(&ss.ready, cudaEventDisableTiming));
        VK_CUDA(cudaEventRecord(ss.ready, st));
        sampler_add_reader(s, st);  // the exchange read the sampler's all-vertex lists
        ss.prefetched = run;
        return;
      }
    }
    const dim3 grid((unsigned)std::max<std::uint64_t>(1, units));
    auto launch = [&](auto tag) {
      using T = decltype(tag);
      const bool fix = gp.V > kMagicExactV;
      if (staged)
        fix ? k_gather<T, true, true><<<grid, 256, 0, st>>>(gp) : k_gather<T, true, false><<<grid, 256, 0, st>>>(gp);
      else
        fix ? k_gather<T, false, true><<<grid, 256, 0, st>>>(gp) : k_gather<T, false, false><<<grid, 256, 0, st>>>(gp);
    };
    if (v16)
      launch(uint4{});
    else if (v4)
      launch(std::uint32_t{});
    else
      launch(std::uint16_t{});
    count_launch();
    VK_LAUNCH_CHECK();
    sampler_add_reader(s, st);  // the next run of this sampler waits for this gather
  }
}

}  // namespace

extern "C" {

int vk_plane_gather(vk_plane p, vk_sampler s, void* out_dev, uint64_t out_stride_rows, uint64_t* counts_dev,
                    vk_stream_t stream) {
  return guard([&] { gather_impl(p, s, out_dev, out_stride_rows, counts_dev, stream, false); });
}

int vk_plane_prefetch(vk_plane p, vk_sampler s) {
  return guard([&] { gather_impl(p, s, nullptr, 0, nullptr, nullptr, true); });
}

int vk_plane_prefetch_after(vk_plane p, vk_sampler s, vk_stream_t after) {
  return guard([&] {
    if (!p) raise(VK_ERR_PARAMETER, "null plane");
    if (after) {
      DeviceGuard dg(p->device);
      VK_CUDA(cudaEventRecord(p->after_ev, static_cast<cudaStream_t>(after)));
      VK_CUDA(cudaStreamWaitEvent(p->aux, p->after_ev, 0));
    }
    gather_impl(p, s, nullptr, 0, nullptr, nullptr, true);
  });
}

}  // extern "C"
