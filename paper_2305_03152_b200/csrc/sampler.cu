// Node-wise fanout sampler on the device, bit-identical to vipkit::expand
// (/root/reference/proj/src/sampling.cpp:72-128), batched over a "wave" of
// minibatches so one launch keeps the whole GPU busy.
//
// Per hop h = 1..L, for every minibatch of the wave:
//   k_sample   one thread per vertex v of F_{h-1}: stream key =
//              key_step(prefix(e,k,i,h), v) (sampling.cpp:110-112); deg <= f
//              copies the CSR slice, else a *sparse* partial Fisher-Yates over
//              the neighbour list (positions < f tracked in a small array,
//              displaced positions >= f in a <= f-entry map) -- the same draw
//              sequence as the reference's full scratch copy (sampling.cpp:
//              82-91), verified in tests. Draws land at the source's MFG row
//              (indptr) and set bits in the hop bitmap and the all bitmap.
//   k_compact  single-pass decoupled look-back over the hop bitmap:
//              F_h = sorted distinct ids (sort+unique of sampling.cpp:115-116
//              for free), per-word rank prefix, and -- fused -- the next hop's
//              MFG indptr = exclusive scan of min(f_{h+1}, deg(v)).
//   k_relabel  MFG dst = rank of each drawn id in F_h (bitmap rank: prefix
//              word + popc).
// Then all_vertices = compaction of the all bitmap (sampling.cpp:121-126) and
// the relabel map F_h -> index in all_vertices.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "rng.cuh"
#include "scan.cuh"

namespace vk {

constexpr int kCompactThreads = 256;
constexpr int kTileWords = kCompactThreads;  // one 64-bit word per thread

// Per-minibatch wave descriptor (uploaded once per run).
struct WaveDesc {
  std::uint64_t key_prefix[VK_MAX_HOPS];
  std::uint64_t seed_begin;
  std::uint32_t seed_count;
  std::uint32_t partition;
};

}  // namespace vk
using vk::WaveDesc;
using vk::kCompactThreads;
using vk::kTileWords;

struct vk_sampler_s {
  vk_graph_s* g = nullptr;
  vk_sampler_config cfg{};
  std::uint32_t L = 0, M = 0;
  std::uint64_t n = 0, W = 0, tiles = 0;
  std::uint64_t capF[VK_MAX_HOPS + 1]{};  // [0] = batch size
  std::uint64_t capS[VK_MAX_HOPS + 1]{};  // [h] edges of hop h
  std::uint64_t capS_max = 0, capAll = 0;
  // all-level rank words written for every word (not only nonzero ones) when
  // that costs no more than the id list itself (16 W <= 4 capAll): the plane
  // then derives the wave's remote-miss set from the bitmaps word by word
  bool dense_all_rank = false;
  // sparse frontiers (frontier_sparse.cuh): bucket bits per level ([0] = all
  // level, [h] = hop h), bucket workspaces sized for the largest level
  bool sparse = false;
  std::uint32_t bb[VK_MAX_HOPS + 1]{};
  std::uint32_t nb_max = 0;
  std::uint64_t pair_stride = 0;
  vk::DevBuf bhist, bstart, bcursor, bstatus, pairs, tile_base, fbase;  // fbase: [L+1][M][NB+1] hop bucket bases
  std::uint32_t nbuckets(std::uint32_t level) const { return (std::uint32_t)((n + (1ull << bb[level]) - 1) >> bb[level]); }
  vk::DevBuf F[VK_MAX_HOPS + 1], allidx[VK_MAX_HOPS + 1], indptr[VK_MAX_HOPS + 1], dst[VK_MAX_HOPS + 1];
  vk::DevBuf counts;  // u32: fcount[(L+1)*M] | ecount[(L+1)*M] | allcount[M] | err[1]
  vk::DevBuf edges_tmp, all, hopbits, allbits, hopprefix, allprefix, status, tickets, desc, seed_stage;
  // pinned staging ring for host seeds / wave descriptors: the host may run
  // kStageSlots - 1 waves ahead of the device
  static constexpr int kStageSlots = 4;
  vk::PinnedBuf desc_host[kStageSlots], seed_host[kStageSlots];
  cudaEvent_t staged[kStageSlots] = {};
  bool staged_used[kStageSlots] = {};
  int slot = 0;
  std::uint32_t last_nmb = 0;
  std::vector<std::uint32_t> last_parts;
  cudaEvent_t done = nullptr;
  // readers of the last run on other streams (a plane gather, its miss
  // exchange on the plane's aux stream): the next run waits for them before
  // it rewrites the workspace they read
  std::vector<cudaEvent_t> readers, reader_pool;
  cudaStream_t stream = nullptr;
  cudaStream_t last_stream = nullptr;
  // seed_keys replay (sampling.hpp:46-56): per-vertex stream keys and a copy
  // of the CSR with every row ordered by key (sample_neighbors' sorted
  // scratch, sampling.cpp:83-85)
  vk::DevBuf keys, tgt_keyed;
  bool keyed = false;
  std::uint64_t runs = 0;  // completed vk_sampler_run calls (plane prefetch bookkeeping)
  // the MFG relabel of hop h runs on `aux` while the main stream samples hop
  // h+1 (or compacts the all level after the last hop); sampled edges are
  // double-buffered by hop parity in edges_tmp
  cudaStream_t aux = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  std::uint32_t* edges_buf(std::uint32_t h) const {
    return edges_tmp.as<std::uint32_t>() + (std::uint64_t)(h & 1u) * M * capS_max;
  }

  std::uint32_t* fcount(std::uint32_t h) const { return counts.as<std::uint32_t>() + (std::uint64_t)h * M; }
  std::uint32_t* ecount(std::uint32_t h) const {
    return counts.as<std::uint32_t>() + (std::uint64_t)(L + 1) * M + (std::uint64_t)h * M;
  }
  std::uint32_t* allcount() const { return counts.as<std::uint32_t>() + 2ull * (L + 1) * M; }
  std::uint32_t* err() const { return allcount() + M; }
  std::size_t counts_words() const { return 2ull * (L + 1) * M + M + 1; }
};

namespace vk {
namespace {

// ------------------------------------------------------------- kernels

// Hop-1 preparation, one CTA per minibatch: copy the seeds into F_0, mark
// them in the all bitmap, and scan min(f_1, deg) into the hop-1 indptr.
__global__ void __launch_bounds__(1024) k_prepare(const WaveDesc* __restrict__ desc,
                                                  const std::uint32_t* __restrict__ seeds,
                                                  const std::uint32_t* __restrict__ outdeg, std::uint64_t n,
                                                  std::uint32_t f1, std::uint32_t* __restrict__ F0,
                                                  std::uint64_t capF0, std::uint32_t* __restrict__ fcount0,
                                                  std::uint32_t* __restrict__ indptr1,
                                                  std::uint32_t* __restrict__ ecount1,
                                                  unsigned long long* __restrict__ allbits, std::uint64_t W,
                                                  std::uint32_t* __restrict__ err) {
  __shared__ unsigned long long sm[32];
  const std::uint32_t mb = blockIdx.x;
  const WaveDesc d = desc[mb];
  std::uint32_t* f0 = F0 + mb * capF0;
  std::uint32_t* ip = indptr1 + mb * (capF0 + 1);
  unsigned long long* ab = allbits ? allbits + mb * W : nullptr;
  unsigned long long carry = 0;
  for (std::uint32_t base = 0; base < d.seed_count; base += blockDim.x) {
    const std::uint32_t i = base + threadIdx.x;
    unsigned long long c = 0;
    if (i < d.seed_count) {
      std::uint32_t v = seeds[d.seed_begin + i];
      if (v >= n) {
        atomicOr(err, 1u);
        v = 0;
      }
      f0[i] = v;
      if (ab) atomicOr(ab + (v >> 6), 1ull << (v & 63));
      c = min(f1, outdeg[v]);
    }
    unsigned long long tot;
    const unsigned long long inc = block_inclusive_scan<1024>(c, sm, &tot);
    if (i < d.seed_count) ip[i] = (std::uint32_t)(carry + inc - c);
    carry += tot;
  }
  if (threadIdx.x == 0) {
    ip[d.seed_count] = (std::uint32_t)carry;
    ecount1[mb] = (std::uint32_t)carry;
    fcount0[mb] = d.seed_count;
  }
}

// Frontier bitmap insert: a 32-bit RED on the half of the 64-bit word that
// holds v (little-endian halves), no return value.
__device__ __forceinline__ void set_bit(unsigned long long* hb, std::uint32_t v) {
  if (hb) atomicOr(reinterpret_cast<unsigned*>(hb) + (v >> 5), 1u << (v & 31));  // null: sparse frontiers
}

// Sparse partial Fisher-Yates, same draws as sampling.cpp:87-91: the value
// at positions [0, f) lives in lo[], positions >= f displaced by a swap in the
// (hp, hv) map (at most f entries); untouched positions read the CSR slice.
// `S` is the slot stride of the per-thread arrays (blockDim for the shared-
// memory layout, where thread t's slot i is at i*S + t, bank-conflict free;
// 1 for the local-memory fallback used for fanouts > 32).
__device__ __forceinline__ void sample_one(const std::uint32_t* __restrict__ nbrs, std::uint32_t deg,
                                           std::uint32_t f, Stream& s, std::uint32_t* __restrict__ out,
                                           unsigned long long* __restrict__ hb, std::uint32_t* lo,
                                           std::uint32_t* hp, std::uint32_t* hv, unsigned S) {
  if (deg <= f) {  // sampling.cpp:76-78: all neighbours, CSR order
    for (std::uint32_t i = 0; i < deg; ++i) {
      const std::uint32_t u = __ldg(nbrs + i);
      out[i] = u;
      set_bit(hb, u);
    }
    return;
  }
  for (std::uint32_t i = 0; i < f; ++i) lo[i * S] = __ldg(nbrs + i);
  std::uint32_t nh = 0;
  for (std::uint32_t i = 0; i < f; ++i) {
    const std::uint32_t j = i + (std::uint32_t)s.next_below((std::uint64_t)(deg - i));
    const std::uint32_t vi = lo[i * S];
    std::uint32_t vj;
    if (j < f) {
      vj = lo[j * S];
      lo[j * S] = vi;
    } else {
      std::uint32_t c = 0;
      while (c < nh && hp[c * S] != j) ++c;
      if (c < nh) {
        vj = hv[c * S];
        hv[c * S] = vi;
      } else {
        vj = __ldg(nbrs + j);
        hp[nh * S] = j;
        hv[nh * S] = vi;
        ++nh;
      }
    }
    out[i] = vj;  // scratch[i] after the swap
    set_bit(hb, vj);
  }
}

struct SampleParams {
  const WaveDesc* desc;
  std::uint32_t h, f;
  const std::uint64_t* off;
  const std::uint32_t* tgt;
  const std::uint32_t* outdeg;
  const std::uint32_t* Fprev;
  std::uint64_t capFprev;
  const std::uint32_t* fcount_prev;
  const std::uint32_t* indptr;
  std::uint32_t* edges;
  std::uint64_t capS;
  unsigned long long* hopbits;
  std::uint64_t W;
  // vertex-tile schedule (hops >= 2, sources sorted): CTA b serves minibatch
  // b % nmb and the sources inside vertex tile b / nmb, found from the
  // previous hop's rank words; minibatch-fastest order makes the CSR rows of a
  // vertex range L2-resident for every minibatch that samples from them.
  const uint4* rank_prev;
  std::uint32_t nmb, tile_words;
  // seed_keys replay (null: keys are the vertex ids, rows in CSR order)
  const std::uint32_t* keys;
  const std::uint32_t* tgt_keyed;
};

// The stream key of v and the row the partial Fisher-Yates draws from
// (sampling.cpp:108-112 and 83-85; CSR order when not replaying keys).
__device__ __forceinline__ std::uint64_t vertex_key(const SampleParams& p, std::uint32_t v) {
  return p.keys ? (std::uint64_t)__ldg(p.keys + v) : (std::uint64_t)v;
}
__device__ __forceinline__ const std::uint32_t* draw_row(const SampleParams& p, std::uint32_t v, std::uint64_t o0) {
  return (p.keys ? p.tgt_keyed : p.tgt) + o0;
}

// One thread per frontier vertex; FY state in shared memory (f <= 32) or in
// local memory (MAXF > 0, large fanouts).
constexpr int kSampleThreads = 128;
constexpr std::uint64_t kRankStride = 64;  // rank words always written at multiples of this
constexpr std::uint32_t kSampleTileWords = 64;  // 4096 source vertices per (tile, minibatch) CTA

// Register-resident sparse Fisher-Yates for fanouts <= FMAX (compile time):
// the f draws are made first (they depend only on the counter stream), the
// neighbour values at the drawn positions are loaded with independent loads,
// then the swaps are replayed on register arrays -- data-dependent indices
// become unrolled compare/selects instead of dependent shared-memory round
// trips. Same draw sequence as sampling.cpp:87-91.
template <int FMAX>
__device__ __forceinline__ void fy_registers(const std::uint32_t* __restrict__ nbrs, std::uint32_t deg,
                                             std::uint32_t f, Stream& s, std::uint32_t* out,
                                             unsigned long long* __restrict__ hb) {
  std::uint32_t jj[FMAX], lo[FMAX], pv[FMAX], hp[FMAX], hv[FMAX];
#pragma unroll
  for (int i = 0; i < FMAX; ++i) jj[i] = (std::uint32_t)i < f ? i + (std::uint32_t)s.next_below((std::uint64_t)(deg - i)) : 0u;
#pragma unroll
  for (int i = 0; i < FMAX; ++i) {
    lo[i] = (std::uint32_t)i < f ? __ldg(nbrs + i) : 0u;
    pv[i] = ((std::uint32_t)i < f && jj[i] >= f) ? __ldg(nbrs + jj[i]) : 0u;
    hp[i] = 0xffffffffu;
    hv[i] = 0u;
  }
  std::uint32_t nh = 0;
#pragma unroll
  for (int i = 0; i < FMAX; ++i) {
    if ((std::uint32_t)i < f) {
      const std::uint32_t ji = jj[i];
      const std::uint32_t vi = lo[i];
      std::uint32_t vj = 0;
      if (ji < f) {
#pragma unroll
        for (int q = i; q < FMAX; ++q)
          if ((std::uint32_t)q == ji) {
            vj = lo[q];
            lo[q] = vi;
          }
      } else {
        bool found = false;
        // at most i displaced positions exist before step i
#pragma unroll
        for (int c = 0; c < i; ++c)
          if (hp[c] == ji) {
            vj = hv[c];
            hv[c] = vi;
            found = true;
          }
        if (!found) {
          vj = pv[i];  // untouched position: the original CSR value
#pragma unroll
          for (int c = 0; c <= i; ++c)
            if ((std::uint32_t)c == nh) {
              hp[c] = ji;
              hv[c] = vi;
            }
          ++nh;
        }
      }
      out[i] = vj;
      set_bit(hb, vj);
    }
  }
}

// Shared-memory sampler (every fanout <= 32). Per thread, in slot-major
// shared arrays (thread t's slot i at i*kSampleThreads + t, conflict free):
//   lo[f] values at positions [0, f), hp/hv[f] the displaced-position map,
//   jj[f] the draw targets, pv[f] the prefetched CSR values at jj.
// The f draws depend only on the counter stream, so all of them are drawn
// first and their neighbour loads issued in groups of 4 independent loads
// (memory-level parallelism instead of one dependent load per draw); the
// Fisher-Yates swaps are then replayed in order on shared memory. Outputs of a
// warp's 32 consecutive sources are contiguous in the MFG edge array, so they
// are staged per warp and written back with coalesced stores.
// EXACT: the fanout equals FMAX at compile time (the common 5/10/15), so the
// register Fisher-Yates unrolls to exactly f slots with no predication.
template <int FMAX, bool EXACT = false>
__global__ void __launch_bounds__(kSampleThreads) k_sample_smem(SampleParams p) {
  extern __shared__ std::uint32_t sm_fy[];
  constexpr unsigned S = kSampleThreads;
  const unsigned f = EXACT ? (unsigned)FMAX : p.f;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // shared FY slots only for the FMAX == 0 (fanout 17..32) variant
  constexpr unsigned kSlots = FMAX == 0 ? 5 : 0;
  std::uint32_t* lo = sm_fy + threadIdx.x;
  std::uint32_t* hp = lo + f * S;
  std::uint32_t* hv = hp + f * S;
  std::uint32_t* jj = hv + f * S;
  std::uint32_t* pv = jj + f * S;
  std::uint32_t* stage = sm_fy + kSlots * f * S + warp * 32 * f;
  std::uint32_t mb, hi, jstart, jstride;
  if (p.rank_prev) {
    mb = blockIdx.x % p.nmb;
    const std::uint32_t tile = blockIdx.x / p.nmb;
    const std::uint32_t cnt = p.fcount_prev[mb];
    const uint4* rk = p.rank_prev + mb * p.W;
    const std::uint64_t w0 = (std::uint64_t)tile * p.tile_words, w1 = w0 + p.tile_words;
    const std::uint32_t first = w0 < p.W ? rk[w0].z : cnt;
    hi = w1 < p.W ? rk[w1].z : cnt;
    jstart = first + warp * 32;
    jstride = S;
  } else {
    mb = blockIdx.y;
    hi = p.fcount_prev[mb];
    jstart = (blockIdx.x * (S / 32) + warp) * 32;
    jstride = gridDim.x * S;
  }
  const std::uint32_t cnt = hi;
  const std::uint64_t prefix = p.desc[mb].key_prefix[p.h - 1];
  const std::uint32_t* fp = p.Fprev + mb * p.capFprev;
  const std::uint32_t* ip = p.indptr + mb * (p.capFprev + 1);
  std::uint32_t* ed = p.edges + mb * p.capS;
  unsigned long long* hb = p.hopbits ? p.hopbits + mb * p.W : nullptr;
  for (std::uint32_t j0 = jstart; j0 < cnt; j0 += jstride) {
    const std::uint32_t j = j0 + lane;
    const std::uint32_t base = ip[j0];
    if (j < cnt) {
      const std::uint32_t v = fp[j];
      // degree from the two offsets (same 128 B line but at line ends): one
      // random DRAM burst per source instead of a second one into outdeg
      const std::uint64_t o0 = __ldg(p.off + v), o1 = __ldg(p.off + v + 1);
      const std::uint32_t deg = (std::uint32_t)(o1 - o0);
      const std::uint32_t* nbrs = p.tgt + o0;  // CSR order (the deg <= f case)
      std::uint32_t* out = stage + (ip[j] - base);
      if (deg <= f) {  // sampling.cpp:76-78: all neighbours, CSR order
        for (std::uint32_t i0 = 0; i0 < deg; i0 += 4) {
          std::uint32_t t[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) t[u] = i0 + u < deg ? __ldg(nbrs + i0 + u) : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i0 + u < deg) {
              out[i0 + u] = t[u];
              set_bit(hb, t[u]);
            }
        }
      } else if constexpr (FMAX > 0) {
        Stream s(key_step(prefix, vertex_key(p, v)));
        fy_registers<FMAX>(draw_row(p, v, o0), deg, f, s, out, hb);
      } else {
        Stream s(key_step(prefix, vertex_key(p, v)));
        nbrs = draw_row(p, v, o0);
        for (std::uint32_t i = 0; i < f; ++i) jj[i * S] = i + (std::uint32_t)s.next_below((std::uint64_t)(deg - i));
        for (std::uint32_t i0 = 0; i0 < f; i0 += 4) {
          std::uint32_t a[4], b[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const std::uint32_t i = i0 + u;
            const std::uint32_t ji = i < f ? jj[i * S] : 0u;
            a[u] = i < f ? __ldg(nbrs + i) : 0u;
            b[u] = (i < f && ji >= f) ? __ldg(nbrs + ji) : 0u;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i0 + u < f) {
              lo[(i0 + u) * S] = a[u];
              pv[(i0 + u) * S] = b[u];
            }
        }
        std::uint32_t nh = 0;
        for (std::uint32_t i = 0; i < f; ++i) {
          const std::uint32_t ji = jj[i * S];
          const std::uint32_t vi = lo[i * S];
          std::uint32_t vj;
          if (ji < f) {
            vj = lo[ji * S];
            lo[ji * S] = vi;
          } else {
            std::uint32_t c = 0;
            while (c < nh && hp[c * S] != ji) ++c;
            if (c < nh) {
              vj = hv[c * S];
              hv[c * S] = vi;
            } else {
              vj = pv[i * S];  // untouched position: the original CSR value
              hp[nh * S] = ji;
              hv[nh * S] = vi;
              ++nh;
            }
          }
          out[i] = vj;  // scratch[i] after the swap (sampling.cpp:87-91)
          set_bit(hb, vj);
        }
      }
    }
    __syncwarp();
    const std::uint32_t last = min(j0 + 32u, cnt);
    const std::uint32_t total = ip[last] - base;
    for (std::uint32_t i = lane; i < total; i += 32) ed[base + i] = stage[i];
    __syncwarp();
  }
}

// Local-memory fallback for fanouts > 32 (per-thread arrays, direct stores).
template <int MAXF>
__global__ void __launch_bounds__(256) k_sample(SampleParams p) {
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t cnt = p.fcount_prev[mb];
  const std::uint64_t prefix = p.desc[mb].key_prefix[p.h - 1];
  const std::uint32_t* fp = p.Fprev + mb * p.capFprev;
  const std::uint32_t* ip = p.indptr + mb * (p.capFprev + 1);
  std::uint32_t* ed = p.edges + mb * p.capS;
  unsigned long long* hb = p.hopbits ? p.hopbits + mb * p.W : nullptr;
  for (std::uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += gridDim.x * blockDim.x) {
    const std::uint32_t v = fp[j];
    Stream s(key_step(prefix, vertex_key(p, v)));
    std::uint32_t lo[MAXF], hp[MAXF], hv[MAXF];
    const std::uint64_t o0 = p.off[v];
    const std::uint32_t deg = (std::uint32_t)(p.off[v + 1] - o0);
    sample_one(deg <= p.f ? p.tgt + o0 : draw_row(p, v, o0), deg, p.f, s, ed + ip[j], hb, lo, hp, hv, 1);
  }
}

// seed_keys replay: (row, key of target) pairs, warp per row, so one radix
// sort orders every row by key (sample_neighbors' scratch sort).
__global__ void k_keyed_pairs(const std::uint64_t* __restrict__ off, const std::uint32_t* __restrict__ tgt,
                              const std::uint32_t* __restrict__ keys, std::uint64_t n,
                              std::uint64_t* __restrict__ kout, std::uint32_t* __restrict__ vout) {
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t w0 = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) >> 5;
  const std::uint64_t nw = ((std::uint64_t)gridDim.x * blockDim.x) >> 5;
  for (std::uint64_t u = w0; u < n; u += nw)
    for (std::uint64_t i = off[u] + lane; i < off[u + 1]; i += 32) {
      const std::uint32_t t = __ldg(tgt + i);
      kout[i] = (u << 32) | __ldg(keys + t);
      vout[i] = t;
    }
}

struct CompactParams {
  unsigned long long* bits;        // [M][W]; zeroed as it is consumed (clean for the next hop/wave)
  unsigned long long* allbits;     // hop compactions OR their words into the all bitmap
  std::uint32_t* list;             // [M][cap_list]
  std::uint64_t cap_list;
  uint4* rank;                     // [M][W] {bits lo, bits hi, rank prefix, 0} per word
  std::uint32_t* count;            // [M]
  // fused next-hop indptr (has_next)
  const std::uint32_t* outdeg;
  std::uint32_t f_next;
  std::uint32_t* indptr_next;      // [M][cap_list + 1]
  std::uint32_t* ecount_next;      // [M]
  unsigned long long* status;      // [M][tiles]
  unsigned* ticket;
  std::uint64_t W, tiles;
  std::uint32_t nmb, wpt;
  std::uint32_t dense_rank;        // write every rank word (see vk_sampler_s::dense_all_rank)
};

constexpr int kStage = 5120;  // ids staged in shared memory per tile (else direct writes)

// One word (64 vertices) per thread, one tile of kTileWords words per CTA.
// Tile ids are emitted into shared memory at their scanned positions and
// copied out with coalesced stores (direct scattered stores only for the rare
// tile denser than kStage).
// Degrees min(f, deg(v)) of the set bits of one word, loads 8 in flight.
__device__ __forceinline__ unsigned long long capped_degree_sum(unsigned long long x, std::uint64_t w,
                                                                const std::uint32_t* __restrict__ outdeg,
                                                                std::uint32_t f) {
  unsigned long long dc = 0;
  while (x) {
    std::uint32_t d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      d[q] = 0;
      if (x) {
        const int b = __ffsll(x) - 1;
        x &= x - 1;
        d[q] = __ldg(outdeg + (std::uint32_t)(w * 64 + b));
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) dc += min(f, d[q]);
  }
  return dc;
}

}  // namespace
}  // namespace vk
#include "frontier_sparse.cuh"
namespace vk {
namespace {

// Narrow tiles (<= 4 words/thread): words held in registers, fully unrolled.
template <bool HAS_NEXT, bool OR_ALL, int WPT>
__global__ void __launch_bounds__(kCompactThreads) k_compact_reg(CompactParams p) {
  constexpr std::uint64_t TW = (std::uint64_t)kCompactThreads * WPT;  // words per tile
  __shared__ unsigned s_ticket;
  __shared__ unsigned long long s_sm[kCompactThreads / 32];
  __shared__ unsigned long long s_excl;
  __shared__ std::uint32_t s_ids[kStage];
  __shared__ std::uint32_t s_ip[HAS_NEXT ? kStage : 1];
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1u);
  __syncthreads();
  const unsigned ticket = s_ticket;
  const std::uint32_t mb = ticket / (unsigned)p.tiles;
  const std::uint32_t tile = ticket % (unsigned)p.tiles;
  if (mb >= p.nmb) return;
  unsigned long long* bits = p.bits + mb * p.W;
  const std::uint64_t w0 = (std::uint64_t)tile * TW + (std::uint64_t)threadIdx.x * WPT;
  unsigned long long wd[WPT];
#pragma unroll
  for (int k = 0; k < WPT; ++k) wd[k] = w0 + k < p.W ? bits[w0 + k] : 0ull;
  unsigned long long vc = 0, dc = 0;
#pragma unroll
  for (int k = 0; k < WPT; ++k) {
    if (wd[k]) {
      bits[w0 + k] = 0ull;  // the rank array keeps the bits; the bitmap is clean for reuse
      if (OR_ALL) atomicOr(p.allbits + mb * p.W + w0 + k, wd[k]);  // RED: no load latency
    }
    vc += __popcll(wd[k]);
    if (HAS_NEXT) {
      // next-hop row lengths min(f, deg): degree loads issued 8 at a time
      unsigned long long x = wd[k];
      while (x) {
        std::uint32_t d[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          d[q] = 0;
          if (x) {
            const int b = __ffsll(x) - 1;
            x &= x - 1;
            d[q] = __ldg(p.outdeg + (std::uint32_t)((w0 + k) * 64 + b));
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) dc += min(p.f_next, d[q]);
      }
    }
  }
  const unsigned long long mine = pack_vd(vc, dc);
  unsigned long long total;
  const unsigned long long inc = block_inclusive_scan<kCompactThreads>(mine, s_sm, &total);
  const unsigned long long lex = inc - mine;  // tile-local exclusive prefix
  const std::uint32_t tcount = (std::uint32_t)unpack_v(total);
  std::uint32_t* list = p.list + mb * p.cap_list;
  std::uint32_t* ipn = HAS_NEXT ? p.indptr_next + mb * (p.cap_list + 1) : nullptr;
  unsigned long long* status = p.status + mb * p.tiles;
  const bool staged = tcount <= (std::uint32_t)kStage;
  // Emit this thread's ids (and next-hop row starts) at positions lpos,
  // dpos; to shared memory at tile-local positions when staged, else
  // directly to the global list.
  auto emit = [&](std::uint32_t lpos, std::uint32_t dpos, std::uint32_t gbase, bool to_smem) {
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
      const std::uint64_t w = w0 + k;
      unsigned long long x = wd[k];
      while (x) {
        // up to 8 set bits per round; their degree loads are independent
        std::uint32_t vv[8], dd[8];
        int nq = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          dd[q] = 0;
          if (x) {
            const int b = __ffsll(x) - 1;
            x &= x - 1;
            vv[q] = (std::uint32_t)(w * 64 + b);
            if (HAS_NEXT) dd[q] = __ldg(p.outdeg + vv[q]);
            nq = q + 1;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < nq) {
            const std::uint32_t v = vv[q];
            std::uint32_t d = 0;
            if (HAS_NEXT) {
              d = dpos;
              dpos += min(p.f_next, dd[q]);
            }
            if (to_smem) {
              s_ids[lpos] = v;
              if (HAS_NEXT) s_ip[lpos] = d;
            } else {
              list[gbase + lpos] = v;
              if (HAS_NEXT) ipn[gbase + lpos] = d;
            }
            ++lpos;
          }
        }
      }
    }
  };
  // rank words are only ever read for set bits (relabel / relabel maps) and
  // at tile starts (multiples of kRankStride words, the vertex-tile
  // schedules): zero words elsewhere are skipped (unless dense_rank), which
  // keeps sparse frontiers on huge graphs from paying 16 B per empty word
  auto write_rank = [&](std::uint32_t first) {
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
      const std::uint64_t w = w0 + k;
      if (w < p.W && (wd[k] || p.dense_rank || (w % kRankStride) == 0))
        p.rank[mb * p.W + w] = make_uint4((unsigned)wd[k], (unsigned)(wd[k] >> 32), first, 0u);
      first += (std::uint32_t)__popcll(wd[k]);
    }
  };
  unsigned long long base;
  if (staged) {
    // ids go to shared memory at tile-local positions first; warp 0 resolves
    // the look-back afterwards, so its latency overlaps the emission (the
    // aggregate is published up front for the successors)
    if (threadIdx.x == 0) publish_aggregate(status, tile, total);
    emit((std::uint32_t)unpack_v(lex), (std::uint32_t)unpack_d(lex), 0u, true);
    if (threadIdx.x < 32) {
      const unsigned long long ex = lookback_resolve(status, tile, total);
      if (threadIdx.x == 0) s_excl = ex;
    }
    __syncthreads();
    base = s_excl;
    const std::uint32_t gbase = (std::uint32_t)unpack_v(base), dbase = (std::uint32_t)unpack_d(base);
    write_rank(gbase + (std::uint32_t)unpack_v(lex));
    for (std::uint32_t i = threadIdx.x; i < tcount; i += kCompactThreads) {
      list[gbase + i] = s_ids[i];
      if (HAS_NEXT) ipn[gbase + i] = dbase + s_ip[i];
    }
  } else {
    if (threadIdx.x < 32) {
      const unsigned long long ex = lookback_warp(status, tile, total);
      if (threadIdx.x == 0) s_excl = ex;
    }
    __syncthreads();
    base = s_excl;
    const std::uint32_t gbase = (std::uint32_t)unpack_v(base);
    write_rank(gbase + (std::uint32_t)unpack_v(lex));
    emit((std::uint32_t)unpack_v(lex), (std::uint32_t)(unpack_d(base) + unpack_d(lex)), gbase, false);
  }
  if (tile == p.tiles - 1 && threadIdx.x == kCompactThreads - 1) {
    const unsigned long long all = base + total;
    const std::uint32_t tv = (std::uint32_t)unpack_v(all), td = (std::uint32_t)unpack_d(all);
    p.count[mb] = tv;
    if (HAS_NEXT) {
      ipn[tv] = td;
      p.ecount_next[mb] = td;
    }
  }
}

// Wide tiles (8 or 16 words per thread; sparse frontiers, papers-scale
// graphs): the tile's words are staged through shared memory with coalesced
// loads, each thread notes which of its words are nonzero, and every later
// pass visits only those (plus the rank-stride word), so an empty word costs
// one shared load and a compare.
template <bool HAS_NEXT, bool OR_ALL>
__global__ void __launch_bounds__(kCompactThreads) k_compact(CompactParams p) {
  __shared__ unsigned s_ticket;
  __shared__ unsigned long long s_sm[kCompactThreads / 32];
  __shared__ unsigned long long s_excl;
  __shared__ std::uint32_t s_ids[kStage];
  __shared__ std::uint32_t s_ip[HAS_NEXT ? kStage : 1];
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1u);
  __syncthreads();
  const unsigned ticket = s_ticket;
  const std::uint32_t mb = ticket / (unsigned)p.tiles;
  const std::uint32_t tile = ticket % (unsigned)p.tiles;
  if (mb >= p.nmb) return;
  const unsigned wpt = p.wpt;  // power of two, 8..32
  unsigned long long* bits = p.bits + mb * p.W;
  const std::uint64_t tbase = (std::uint64_t)tile * kCompactThreads * wpt;
  const std::uint64_t w0 = tbase + (std::uint64_t)threadIdx.x * wpt;
  const unsigned nw = w0 < p.W ? (unsigned)min((std::uint64_t)wpt, p.W - w0) : 0u;
  // row pitch wpt+1 avoids bank conflicts; 32-bit shifts, no division
  extern __shared__ unsigned long long s_words[];
  {
    const unsigned n_t = (unsigned)(min(tbase + (std::uint64_t)kCompactThreads * wpt, p.W) - tbase);
    const unsigned lw = (unsigned)(__ffs((int)wpt) - 1);
    const unsigned long long* tb = bits + tbase;
    // wpt (8..32) coalesced rounds, 8 loads in flight per thread before the
    // shared stores (a dependent load->store loop would pay one DRAM latency
    // per round)
    for (unsigned i0 = 0; i0 < wpt; i0 += 8) {
      unsigned long long r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const unsigned o = (i0 + q) * kCompactThreads + threadIdx.x;
        r[q] = o < n_t ? tb[o] : 0ull;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const unsigned o = (i0 + q) * kCompactThreads + threadIdx.x;
        if (o < n_t) s_words[(o >> lw) * (wpt + 1) + (o & (wpt - 1))] = r[q];
      }
    }
    __syncthreads();
  }
  const unsigned long long* my = s_words + threadIdx.x * (wpt + 1);
  unsigned nz = 0;
  unsigned long long vc = 0, dc = 0;
  for (unsigned j = 0; j < nw; ++j) {
    const unsigned long long wd = my[j];
    if (wd) {
      nz |= 1u << j;
      vc += __popcll(wd);
    }
  }
  // Cursor over this thread's set bits in vertex order, across its nonzero
  // words: sparse tiles have ~1 bit per word, so gathering 8 bits per round
  // across words keeps 8 degree loads in flight instead of one per word.
  auto next8 = [&](unsigned& m, unsigned long long& x, unsigned& j, std::uint32_t* vv) -> int {
    int nq = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      while (!x && m) {
        j = (unsigned)(__ffs((int)m) - 1);
        m &= m - 1;
        x = my[j];
      }
      if (x) {
        const int b = __ffsll(x) - 1;
        x &= x - 1;
        vv[q] = (std::uint32_t)((w0 + j) * 64 + b);
        nq = q + 1;
      }
    }
    return nq;
  };
  // the first 8 degrees stay in registers for the emission pass (sparse
  // tiles: every degree; no second random DRAM burst per vertex)
  std::uint32_t cd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) cd[q] = 0u;
  if (HAS_NEXT) {
    unsigned m = nz, j = 0;
    unsigned long long x = 0;
    bool first = true;
    while (true) {
      std::uint32_t vv[8], d[8];
      const int nq = next8(m, x, j, vv);
      if (!nq) break;
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = q < nq ? __ldg(p.outdeg + vv[q]) : 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (first) cd[q] = d[q];
        dc += min(p.f_next, d[q]);
      }
      first = false;
    }
  }
  // words that get a rank entry: nonzero ones, the kRankStride multiple (tile
  // starts of the vertex-tile schedules), or all of them (dense_rank)
  unsigned rmask = nz;
  if (p.dense_rank) {
    rmask = nw >= 32 ? ~0u : ((1u << nw) - 1u);
  } else {
    const unsigned jr = (unsigned)((kRankStride - (w0 % kRankStride)) % kRankStride);
    if (jr < nw) rmask |= 1u << jr;
  }
  const unsigned long long mine = pack_vd(vc, dc);
  unsigned long long total;
  const unsigned long long inc = block_inclusive_scan<kCompactThreads>(mine, s_sm, &total);
  const unsigned long long lex = inc - mine;  // tile-local exclusive prefix
  const std::uint32_t tcount = (std::uint32_t)unpack_v(total);
  std::uint32_t* list = p.list + mb * p.cap_list;
  std::uint32_t* ipn = HAS_NEXT ? p.indptr_next + mb * (p.cap_list + 1) : nullptr;
  unsigned long long* status = p.status + mb * p.tiles;
  const bool staged = tcount <= (std::uint32_t)kStage;
  // Emit this thread's ids (and next-hop row starts) at positions lpos,
  // dpos: to shared memory at tile-local positions, or to the global list.
  auto emit_all = [&](std::uint32_t lpos, std::uint32_t dpos, std::uint32_t gbase, bool to_smem) {
    unsigned m = nz, j = 0;
    unsigned long long x = 0;
    bool first = true;
    while (true) {
      std::uint32_t vv[8], dd[8];
      const int nq = next8(m, x, j, vv);
      if (!nq) break;
#pragma unroll
      for (int q = 0; q < 8; ++q) dd[q] = (HAS_NEXT && q < nq) ? (first ? cd[q] : __ldg(p.outdeg + vv[q])) : 0u;
      first = false;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < nq) {
          std::uint32_t d = 0;
          if (HAS_NEXT) {
            d = dpos;
            dpos += min(p.f_next, dd[q]);
          }
          if (to_smem) {
            s_ids[lpos] = vv[q];
            if (HAS_NEXT) s_ip[lpos] = d;
          } else {
            list[gbase + lpos] = vv[q];
            if (HAS_NEXT) ipn[gbase + lpos] = d;
          }
          ++lpos;
        }
      }
    }
  };
  // Tiles with many nonzero words (>= 1 id per 4 words) clear the whole tile
  // with coalesced stores instead of one partial-sector store per word.
  const bool clear_tile = (std::uint64_t)tcount * 4 >= (std::uint64_t)kCompactThreads * wpt;
  auto finish = [&](std::uint32_t first) {
    for (unsigned m = rmask; m; m &= m - 1) {
      const unsigned j = (unsigned)(__ffs((int)m) - 1);
      const std::uint64_t w = w0 + j;
      const unsigned long long wd = my[j];
      p.rank[mb * p.W + w] = make_uint4((unsigned)wd, (unsigned)(wd >> 32), first, 0u);
      if (wd) {
        if (!clear_tile) bits[w] = 0ull;
        if (OR_ALL) atomicOr(p.allbits + mb * p.W + w, wd);  // RED: no load latency
        first += (std::uint32_t)__popcll(wd);
      }
    }
    if (clear_tile) {
      const unsigned n_t = (unsigned)(min(tbase + (std::uint64_t)kCompactThreads * wpt, p.W) - tbase);
      unsigned long long* tb = bits + tbase;
      for (unsigned o = threadIdx.x; o < n_t; o += kCompactThreads) tb[o] = 0ull;
    }
  };
  unsigned long long base;
  if (staged) {
    // ids to shared memory at tile-local positions first, then warp 0
    // resolves the look-back (its latency overlaps the emission)
    if (threadIdx.x == 0) publish_aggregate(status, tile, total);
    emit_all((std::uint32_t)unpack_v(lex), (std::uint32_t)unpack_d(lex), 0u, true);
    if (threadIdx.x < 32) {
      const unsigned long long ex = lookback_resolve(status, tile, total);
      if (threadIdx.x == 0) s_excl = ex;
    }
    __syncthreads();
    base = s_excl;
    const std::uint32_t gbase = (std::uint32_t)unpack_v(base), dbase = (std::uint32_t)unpack_d(base);
    finish(gbase + (std::uint32_t)unpack_v(lex));
    for (std::uint32_t i = threadIdx.x; i < tcount; i += kCompactThreads) {
      list[gbase + i] = s_ids[i];
      if (HAS_NEXT) ipn[gbase + i] = dbase + s_ip[i];
    }
  } else {
    if (threadIdx.x < 32) {
      const unsigned long long ex = lookback_warp(status, tile, total);
      if (threadIdx.x == 0) s_excl = ex;
    }
    __syncthreads();
    base = s_excl;
    const std::uint32_t gbase = (std::uint32_t)unpack_v(base);
    finish(gbase + (std::uint32_t)unpack_v(lex));
    emit_all((std::uint32_t)unpack_v(lex), (std::uint32_t)(unpack_d(base) + unpack_d(lex)), gbase, false);
  }
  if (tile == p.tiles - 1 && threadIdx.x == kCompactThreads - 1) {
    const unsigned long long all = base + total;
    const std::uint32_t tv = (std::uint32_t)unpack_v(all), td = (std::uint32_t)unpack_d(all);
    p.count[mb] = tv;
    if (HAS_NEXT) {
      ipn[tv] = td;
      p.ecount_next[mb] = td;
    }
  }
}

// Small graphs (W <= kSmallW words): one CTA per minibatch compacts a whole
// level with the bitmap, its word prefixes in shared memory (no look-back
// chain), writes every rank word, and then answers the rank lookups that
// follow from shared memory instead of L2: this hop's MFG relabel, or at the
// all level the relabel maps of every hop.
constexpr std::uint64_t kSmallW = 8192;  // 524,288 vertices: 16 B of shared memory per word
constexpr int kSmallThreads = 1024;

struct SmallParams {
  CompactParams c;
  // hop level: relabel of this hop's sampled edges into dst
  const std::uint32_t* edges;
  std::uint64_t edges_stride;
  const std::uint32_t* ecount;
  std::uint32_t* dst;
  std::uint64_t dst_stride;
  // all level: relabel maps of hops 0..L
  std::uint32_t L;
  const std::uint32_t* F[VK_MAX_HOPS + 1];
  std::uint64_t capF[VK_MAX_HOPS + 1];
  const std::uint32_t* fcount[VK_MAX_HOPS + 1];
  std::uint32_t* allidx[VK_MAX_HOPS + 1];
};

template <bool HAS_NEXT, bool OR_ALL, bool ALL>
__global__ void __launch_bounds__(kSmallThreads) k_compact_small(SmallParams sp) {
  extern __shared__ unsigned long long s_small[];
  __shared__ unsigned long long s_scan[kSmallThreads / 32];
  const CompactParams& p = sp.c;
  const std::uint64_t W = p.W;
  unsigned long long* bw = s_small;                                // [W] the level's bits
  std::uint32_t* pre = reinterpret_cast<std::uint32_t*>(bw + W);  // [W] rank prefix per word
  const std::uint32_t mb = blockIdx.x;
  unsigned long long* bits = p.bits + mb * W;
  for (std::uint64_t w = threadIdx.x; w < W; w += kSmallThreads) {
    const unsigned long long x = bits[w];
    bw[w] = x;
    if (x) {
      bits[w] = 0ull;  // clean for the next hop / wave
      if (OR_ALL) p.allbits[mb * W + w] |= x;  // this CTA owns the minibatch's words
    }
  }
  __syncthreads();
  // contiguous chunk of words per thread
  const std::uint64_t cpt = (W + kSmallThreads - 1) / kSmallThreads;
  const std::uint64_t w0 = min(W, (std::uint64_t)threadIdx.x * cpt), w1 = min(W, w0 + cpt);
  unsigned long long vc = 0, dc = 0;
  for (std::uint64_t w = w0; w < w1; ++w) {
    const unsigned long long x = bw[w];
    vc += __popcll(x);
    if (HAS_NEXT && x) dc += capped_degree_sum(x, w, p.outdeg, p.f_next);
  }
  const unsigned long long mine = pack_vd(vc, dc);
  unsigned long long total;
  const unsigned long long ex = block_inclusive_scan<kSmallThreads>(mine, s_scan, &total) - mine;
  std::uint32_t lpos = (std::uint32_t)unpack_v(ex), dpos = (std::uint32_t)unpack_d(ex);
  std::uint32_t* list = p.list + mb * p.cap_list;
  std::uint32_t* ipn = HAS_NEXT ? p.indptr_next + mb * (p.cap_list + 1) : nullptr;
  for (std::uint64_t w = w0; w < w1; ++w) {
    unsigned long long x = bw[w];
    pre[w] = lpos;
    p.rank[mb * W + w] = make_uint4((unsigned)x, (unsigned)(x >> 32), lpos, 0u);
    while (x) {
      std::uint32_t vv[8], dd[8];
      int nq = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        dd[q] = 0;
        if (x) {
          const int b = __ffsll(x) - 1;
          x &= x - 1;
          vv[q] = (std::uint32_t)(w * 64 + b);
          if (HAS_NEXT) dd[q] = __ldg(p.outdeg + vv[q]);
          nq = q + 1;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nq) {
          list[lpos] = vv[q];
          if (HAS_NEXT) {
            ipn[lpos] = dpos;
            dpos += min(p.f_next, dd[q]);
          }
          ++lpos;
        }
    }
  }
  if (threadIdx.x == kSmallThreads - 1) {
    const std::uint32_t tv = (std::uint32_t)unpack_v(total), td = (std::uint32_t)unpack_d(total);
    p.count[mb] = tv;
    if (HAS_NEXT) {
      ipn[tv] = td;
      p.ecount_next[mb] = td;
    }
  }
  __syncthreads();
  auto rank_of = [&](std::uint32_t v) {
    const std::uint32_t w = v >> 6;
    return pre[w] + (std::uint32_t)__popcll(bw[w] & ((1ull << (v & 63)) - 1ull));
  };
  if (!ALL) {  // the MFG relabel of this hop (k_relabel)
    const std::uint32_t ne = sp.ecount[mb];
    const std::uint32_t* ed = sp.edges + mb * sp.edges_stride;
    std::uint32_t* dst = sp.dst + mb * sp.dst_stride;
    for (std::uint32_t e = threadIdx.x; e < ne; e += kSmallThreads) dst[e] = rank_of(__ldg(ed + e));
  } else {  // relabel maps of every hop (k_allidx)
    for (std::uint32_t h = 0; h <= sp.L; ++h) {
      const std::uint32_t cnt = sp.fcount[h][mb];
      const std::uint32_t* F = sp.F[h] + mb * sp.capF[h];
      std::uint32_t* ai = sp.allidx[h] + mb * sp.capF[h];
      for (std::uint32_t j = threadIdx.x; j < cnt; j += kSmallThreads) ai[j] = rank_of(__ldg(F + j));
    }
  }
}

// Rank of v in the compacted list: one 16-byte load of {bits, prefix} (one
// L2 sector per lookup instead of two).
__device__ __forceinline__ std::uint32_t bit_rank(const uint4* __restrict__ rank, std::uint32_t v) {
  const uint4 r = __ldg(rank + (v >> 6));
  const unsigned long long bits = (unsigned long long)r.x | ((unsigned long long)r.y << 32);
  return r.z + (std::uint32_t)__popcll(bits & ((1ull << (v & 63)) - 1ull));
}

// Rank lookups with kIlp independent elements in flight per thread.
constexpr int kIlp = 4;

__device__ __forceinline__ void rank_range(const std::uint32_t* __restrict__ in, std::uint32_t* __restrict__ out,
                                           std::uint32_t cnt, const uint4* __restrict__ rk) {
  if ((((std::uintptr_t)in | (std::uintptr_t)out) & 15) == 0) {
    // 16 B-aligned lists: 4 consecutive ids per 128-bit load and store
    const std::uint32_t n4 = cnt / 4;
    const uint4* in4 = reinterpret_cast<const uint4*>(in);
    uint4* out4 = reinterpret_cast<uint4*>(out);
    const std::uint32_t stride = gridDim.x * blockDim.x;
    for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const uint4 v = __ldg(in4 + i);
      out4[i] = make_uint4(bit_rank(rk, v.x), bit_rank(rk, v.y), bit_rank(rk, v.z), bit_rank(rk, v.w));
    }
    for (std::uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride)
      out[i] = bit_rank(rk, __ldg(in + i));
    return;
  }
  const std::uint32_t stride = gridDim.x * blockDim.x;
  for (std::uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < cnt; i0 += kIlp * stride) {
    std::uint32_t v[kIlp];
#pragma unroll
    for (int u = 0; u < kIlp; ++u) {
      const std::uint32_t i = i0 + u * stride;
      v[u] = i < cnt ? __ldg(in + i) : 0u;
    }
    std::uint32_t r[kIlp];
#pragma unroll
    for (int u = 0; u < kIlp; ++u) r[u] = bit_rank(rk, v[u]);
#pragma unroll
    for (int u = 0; u < kIlp; ++u) {
      const std::uint32_t i = i0 + u * stride;
      if (i < cnt) out[i] = r[u];
    }
  }
}

// MFG dst: rank of every drawn id in F_h.
__global__ void __launch_bounds__(256) k_relabel(const std::uint32_t* __restrict__ edges, std::uint64_t in_stride,
                                                 const std::uint32_t* __restrict__ ecount,
                                                 const uint4* __restrict__ rank, std::uint64_t W,
                                                 std::uint32_t* __restrict__ dst, std::uint64_t out_stride) {
  const std::uint32_t mb = blockIdx.y;
  rank_range(edges + mb * in_stride, dst + mb * out_stride, ecount[mb], rank + mb * W);
}

// Relabel map: position of every F_h vertex in all_vertices.
__global__ void __launch_bounds__(256) k_allidx(const std::uint32_t* __restrict__ F, std::uint32_t* __restrict__ idx,
                                                std::uint64_t cap, const std::uint32_t* __restrict__ count,
                                                const uint4* __restrict__ rank, std::uint64_t W) {
  const std::uint32_t mb = blockIdx.y;
  rank_range(F + mb * cap, idx + mb * cap, count[mb], rank + mb * W);
}

__global__ void k_stream_draws(std::uint64_t key, std::uint64_t bound, std::uint64_t count,
                               std::uint64_t* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  Stream s(key);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = bound ? s.next_below(bound) : s.next_u64();
}

template <int MAXF>
void launch_sample(vk_sampler_s& s, std::uint32_t h, std::uint32_t nmb, cudaStream_t st) {
  vk_graph_s& g = *s.g;
  SampleParams p;
  p.desc = s.desc.as<WaveDesc>();
  p.h = h;
  p.f = s.cfg.fanouts[h - 1];
  p.off = g.d_off();
  p.tgt = g.d_tgt();
  p.outdeg = g.out_deg.as<std::uint32_t>();
  p.keys = s.keyed ? s.keys.as<std::uint32_t>() : nullptr;
  p.tgt_keyed = s.keyed ? s.tgt_keyed.as<std::uint32_t>() : nullptr;
  p.Fprev = s.F[h - 1].as<std::uint32_t>();
  p.capFprev = s.capF[h - 1];
  p.fcount_prev = s.fcount(h - 1);
  p.indptr = s.indptr[h].as<std::uint32_t>();
  p.edges = s.edges_buf(h);
  p.capS = s.capS_max;
  p.hopbits = s.sparse ? nullptr : s.hopbits.as<unsigned long long>();
  p.W = s.W;
  if constexpr (MAXF == 0) {
    // 5 FY slots per thread + a 32*f staging row per warp
    const int fmax = p.f <= 8 ? 8 : (p.f <= 16 ? 16 : 0);
    const std::size_t smem = (std::size_t)((fmax ? 0 : 5) * kSampleThreads + kSampleThreads) * p.f * 4;
    p.nmb = nmb;
    auto go = [&](dim3 grid) {
      if (p.f == 5)
        k_sample_smem<5, true><<<grid, kSampleThreads, smem, st>>>(p);
      else if (p.f == 10)
        k_sample_smem<10, true><<<grid, kSampleThreads, smem, st>>>(p);
      else if (p.f == 15)
        k_sample_smem<15, true><<<grid, kSampleThreads, smem, st>>>(p);
      else if (fmax == 8)
        k_sample_smem<8><<<grid, kSampleThreads, smem, st>>>(p);
      else if (fmax == 16)
        k_sample_smem<16><<<grid, kSampleThreads, smem, st>>>(p);
      else
        k_sample_smem<0><<<grid, kSampleThreads, smem, st>>>(p);
    };
    p.tile_words = kSampleTileWords;
    if (h >= 2 && !s.sparse) {
      p.rank_prev = s.hopprefix.as<uint4>();
      // ~512 sources per (tile, minibatch) CTA at full frontier capacity,
      // at least kSampleTileWords words (4096 vertices) per tile
      constexpr std::uint64_t tile_sources = 512;  // 256 / 1024 measured flat
      const std::uint64_t want_tiles = std::max<std::uint64_t>(1, p.capFprev / tile_sources);
      std::uint64_t tw = std::max<std::uint64_t>(kSampleTileWords, (s.W + want_tiles - 1) / want_tiles);
      tw = (tw + kRankStride - 1) / kRankStride * kRankStride;  // tile starts carry rank words
      p.tile_words = (std::uint32_t)tw;
      const std::uint64_t tiles = (s.W + tw - 1) / tw;
      go(dim3((unsigned)(tiles * nmb)));
    } else {
      p.rank_prev = nullptr;
      const unsigned gx = (unsigned)std::min<std::uint64_t>(ceil_div(p.capFprev, kSampleThreads), 8192);
      go(dim3(gx, nmb));
    }
  } else {
    const unsigned gx = (unsigned)std::min<std::uint64_t>(ceil_div(p.capFprev, 256), 4096);
    k_sample<MAXF><<<dim3(gx, nmb), 256, 0, st>>>(p);
  }
}

void run_compact(vk_sampler_s& s, bool hop, std::uint32_t h, std::uint32_t nmb, std::uint32_t slot,
                 cudaStream_t st) {
  CompactParams p{};
  p.bits = (hop ? s.hopbits : s.allbits).as<unsigned long long>();
  p.allbits = s.allbits.as<unsigned long long>();
  p.list = hop ? s.F[h].as<std::uint32_t>() : s.all.as<std::uint32_t>();
  p.cap_list = hop ? s.capF[h] : s.capAll;
  p.rank = (hop ? s.hopprefix : s.allprefix).as<uint4>();
  p.count = hop ? s.fcount(h) : s.allcount();
  const bool has_next = hop && h < s.L;
  p.outdeg = s.g->out_deg.as<std::uint32_t>();
  if (has_next) {
    p.f_next = s.cfg.fanouts[h];
    p.indptr_next = s.indptr[h + 1].as<std::uint32_t>();
    p.ecount_next = s.ecount(h + 1);
  }
  p.status = s.status.as<unsigned long long>() + (std::uint64_t)slot * s.M * s.tiles;
  p.ticket = s.tickets.as<unsigned>() + slot;
  p.W = s.W;
  p.nmb = nmb;
  p.dense_rank = (!hop && s.dense_all_rank) ? 1u : 0u;
  // Words per thread from the frontier's expected density (its capacity / n):
  // the widest tile whose expected ids still fit the shared staging buffer.
  // Sparse frontiers (early hops, papers-scale graphs) get few, fat tiles
  // instead of ~W/256 tiny CTAs; the dense C3 last hop keeps 1 word/thread.
  const double density = (double)p.cap_list / (double)std::max<std::uint64_t>(1, s.n);
  int wpt = 1;
  // ... but never fewer than ~8 CTAs per SM in total
  const std::uint64_t min_ctas = (std::uint64_t)sm_count(s.g->device) * 8;
  auto ctas = [&](int w) { return (std::uint64_t)nmb * ((s.W + (std::uint64_t)kCompactThreads * w - 1) /
                                                         ((std::uint64_t)kCompactThreads * w)); };
  constexpr int max_wpt = 16;  // 32 measured no faster
  while (wpt < max_wpt && (double)kCompactThreads * (wpt * 2) * 64.0 * density <= (double)kStage &&
         ctas(wpt * 2) >= min_ctas)
    wpt *= 2;
  p.tiles = (s.W + (std::uint64_t)kCompactThreads * wpt - 1) / ((std::uint64_t)kCompactThreads * wpt);
  const unsigned grid = (unsigned)(nmb * p.tiles);
  p.wpt = (std::uint32_t)wpt;
  const std::size_t smem = wpt >= 8 ? (std::size_t)kCompactThreads * (wpt + 1) * 8 : 0;
  auto narrow = [&](auto hn, auto oa) {
    constexpr bool HN = decltype(hn)::value, OA = decltype(oa)::value;
    if (wpt == 4)
      k_compact_reg<HN, OA, 4><<<grid, kCompactThreads, 0, st>>>(p);
    else if (wpt == 2)
      k_compact_reg<HN, OA, 2><<<grid, kCompactThreads, 0, st>>>(p);
    else
      k_compact_reg<HN, OA, 1><<<grid, kCompactThreads, 0, st>>>(p);
  };
  if (wpt >= 32) {  // 32 words/thread stage 67 KB
    const int mx = (int)smem;
    VK_CUDA(cudaFuncSetAttribute(k_compact<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    VK_CUDA(cudaFuncSetAttribute(k_compact<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    VK_CUDA(cudaFuncSetAttribute(k_compact<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  }
  if (wpt <= 4) {
    if (has_next)
      narrow(std::true_type{}, std::true_type{});
    else if (hop)
      narrow(std::false_type{}, std::true_type{});
    else
      narrow(std::false_type{}, std::false_type{});
  } else if (has_next) {
    k_compact<true, true><<<grid, kCompactThreads, smem, st>>>(p);
  } else if (hop) {
    k_compact<false, true><<<grid, kCompactThreads, smem, st>>>(p);
  } else {
    k_compact<false, false><<<grid, kCompactThreads, smem, st>>>(p);
  }
}

// Sparse frontiers: one level (hop h >= 1, or the all level for h == 0)
// through hist -> scan -> scatter -> dedup (frontier_sparse.cuh).
template <class P>
void launch_smem(void (*kernel)(P), const P& p, dim3 grid, std::size_t smem, cudaStream_t st) {
  if (smem >= 40 * 1024)  // beyond the default 48 KB with the static shared arrays
    VK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kernel<<<grid, kBktThreads, smem, st>>>(p);
}

void run_bucket_level(vk_sampler_s& s, std::uint32_t h, std::uint32_t nmb, cudaStream_t st) {
  const bool all = h == 0;
  BucketParams bp{};
  bp.bb = s.bb[h];
  bp.NB = s.nbuckets(h);
  bp.hist = s.bhist.as<std::uint32_t>();
  bp.bstart = s.bstart.as<std::uint32_t>();
  bp.cursor = s.bcursor.as<std::uint32_t>();
  bp.pairs = s.pairs.as<uint2>();
  bp.pair_stride = s.pair_stride;
  bp.status = s.bstatus.as<unsigned long long>();
  DedupParams dp{};
  dp.nmb = nmb;
  dp.outdeg = s.g->out_deg.as<std::uint32_t>();
  // dedup grid: groups of kMbGroup minibatches (y), buckets ascending with
  // the minibatch fastest inside a group (x); blocks run in index order
  const dim3 grid(kMbGroup * bp.NB, (unsigned)ceil_div(nmb, kMbGroup));
  if (all) {
    // the sorted levels are ranged by the hops' bucket bases; the batch F_0
    // is bucketed like a hop's draws (its scan also resets the look-back)
    bp.L = s.L;
    for (std::uint32_t q = 0; q <= s.L; ++q) {
      bp.F[q] = s.F[q].as<std::uint32_t>();
      bp.capF[q] = s.capF[q];
      bp.fcount[q] = s.fcount(q);
    }
    bp.ids = s.F[0].as<std::uint32_t>();
    bp.ids_stride = s.capF[0];
    bp.count = s.fcount(0);
    k_bucket_hist<<<dim3((unsigned)std::max<std::uint64_t>(1, ceil_div(s.capF[0], kHistItems)), nmb), kBktThreads,
                    bp.NB * 4, st>>>(bp);
    k_bucket_scan<<<nmb, kScanThreads, 0, st>>>(bp);
    k_bucket_scatter<<<dim3((unsigned)std::max<std::uint64_t>(1, ceil_div(s.capF[0], kScatterItems)), nmb),
                       kBktThreads, scatter_smem(bp.NB), st>>>(bp);
    count_launch(3);
    dp.bp = bp;
    dp.list = s.all.as<std::uint32_t>();
    dp.cap_list = s.capAll;
    dp.count = s.allcount();
    for (std::uint32_t q = 0; q <= s.L; ++q) {
      dp.allidx[q] = s.allidx[q].as<std::uint32_t>();
      dp.fbase[q] = s.fbase.as<std::uint32_t>() + (std::uint64_t)q * s.M * (s.nb_max + 1);
    }
    dp.base_out = s.tile_base.as<std::uint32_t>();
    launch_smem(k_bucket_dedup_all, dp, grid, dedup_smem(bp.bb, false), st);
    count_launch();
    VK_LAUNCH_CHECK();
    return;
  }
  bp.ids = s.edges_buf(h);
  bp.ids_stride = s.capS_max;
  bp.count = s.ecount(h);
  if (s.capS[h] <= kSmallLevel) {  // one sorting CTA per minibatch
    dp.bp = bp;
    dp.list = s.F[h].as<std::uint32_t>();
    dp.cap_list = s.capF[h];
    dp.count = s.fcount(h);
    dp.dst = s.dst[h].as<std::uint32_t>();
    dp.dst_stride = s.capS[h];
    dp.base_out = s.fbase.as<std::uint32_t>() + (std::uint64_t)h * s.M * (s.nb_max + 1);
    const std::size_t smem = (std::size_t)kSmallLevel * 8;
    auto go = [&](void (*kernel)(DedupParams)) {
      VK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kernel<<<nmb, kSmallLevelThreads, smem, st>>>(dp);
    };
    if (h < s.L) {
      dp.f_next = s.cfg.fanouts[h];
      dp.indptr_next = s.indptr[h + 1].as<std::uint32_t>();
      dp.ecount_next = s.ecount(h + 1);
      go(k_small_level<true>);
    } else {
      go(k_small_level<false>);
    }
    count_launch();
    VK_LAUNCH_CHECK();
    return;
  }
  k_bucket_hist<<<dim3((unsigned)std::max<std::uint64_t>(1, ceil_div(s.capS[h], kHistItems)), nmb), kBktThreads,
                  bp.NB * 4, st>>>(bp);
  k_bucket_scan<<<nmb, kScanThreads, 0, st>>>(bp);
  k_bucket_scatter<<<dim3((unsigned)std::max<std::uint64_t>(1, ceil_div(s.capS[h], kScatterItems)), nmb),
                     kBktThreads, scatter_smem(bp.NB), st>>>(bp);
  count_launch(3);
  VK_LAUNCH_CHECK();
  dp.bp = bp;
  dp.list = s.F[h].as<std::uint32_t>();
  dp.cap_list = s.capF[h];
  dp.count = s.fcount(h);
  dp.dst = s.dst[h].as<std::uint32_t>();
  dp.dst_stride = s.capS[h];
  dp.base_out = s.fbase.as<std::uint32_t>() + (std::uint64_t)h * s.M * (s.nb_max + 1);
  if (h < s.L) {
    dp.f_next = s.cfg.fanouts[h];
    dp.indptr_next = s.indptr[h + 1].as<std::uint32_t>();
    dp.ecount_next = s.ecount(h + 1);
    launch_smem(k_bucket_dedup_hop<true>, dp, grid, dedup_smem(bp.bb, true), st);
  } else {
    launch_smem(k_bucket_dedup_hop<false>, dp, grid, dedup_smem(bp.bb, false), st);
  }
  count_launch();
  VK_LAUNCH_CHECK();
}

// Bucket bits of a level with `items` items per minibatch at capacity: about
// kBucketTarget items per bucket, 2^14..2^19 ids per bucket (shared bitmap
// of 2..64 KB), at most kMaxBuckets buckets.
std::uint32_t bucket_bits(std::uint64_t n) {
  // 2^14..2^19 ids per bucket (2..64 KB of shared bitmap), at most
  // kMaxBuckets; ~512 buckets per minibatch: C4 (111 M ids) -> 2^18 ids per
  // bucket (measured per C4 wave of 64: 2^17 5.3 ms, 2^18 4.2 ms, 2^19 4.2 ms)
  std::uint32_t bb = (std::uint32_t)std::ceil(std::log2(std::max(1.0, (double)n / 512.0)));
  bb = std::min<std::uint32_t>(18, std::max<std::uint32_t>(14, bb));
  while (bb < 19 && ((n + (1ull << bb) - 1) >> bb) > kMaxBuckets) ++bb;
  return bb;
}

void run_compact_small(vk_sampler_s& s, bool hop, std::uint32_t h, std::uint32_t nmb, cudaStream_t st) {
  SmallParams sp{};
  CompactParams& p = sp.c;
  p.bits = (hop ? s.hopbits : s.allbits).as<unsigned long long>();
  p.allbits = s.allbits.as<unsigned long long>();
  p.list = hop ? s.F[h].as<std::uint32_t>() : s.all.as<std::uint32_t>();
  p.cap_list = hop ? s.capF[h] : s.capAll;
  p.rank = (hop ? s.hopprefix : s.allprefix).as<uint4>();
  p.count = hop ? s.fcount(h) : s.allcount();
  p.outdeg = s.g->out_deg.as<std::uint32_t>();
  const bool has_next = hop && h < s.L;
  if (has_next) {
    p.f_next = s.cfg.fanouts[h];
    p.indptr_next = s.indptr[h + 1].as<std::uint32_t>();
    p.ecount_next = s.ecount(h + 1);
  }
  p.W = s.W;
  p.nmb = nmb;
  if (hop) {
    sp.edges = s.edges_buf(h);
    sp.edges_stride = s.capS_max;
    sp.ecount = s.ecount(h);
    sp.dst = s.dst[h].as<std::uint32_t>();
    sp.dst_stride = s.capS[h];
  } else {
    sp.L = s.L;
    for (std::uint32_t q = 0; q <= s.L; ++q) {
      sp.F[q] = s.F[q].as<std::uint32_t>();
      sp.capF[q] = s.capF[q];
      sp.fcount[q] = s.fcount(q);
      sp.allidx[q] = s.allidx[q].as<std::uint32_t>();
    }
  }
  const std::size_t smem = (std::size_t)s.W * 12;
  static bool attr = false;  // up to 96 KB of dynamic shared memory
  if (!attr) {
    const int mx = (int)(kSmallW * 12);
    VK_CUDA(cudaFuncSetAttribute(k_compact_small<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    VK_CUDA(cudaFuncSetAttribute(k_compact_small<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    VK_CUDA(cudaFuncSetAttribute(k_compact_small<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    attr = true;
  }
  auto go = [&](void (*kernel)(SmallParams)) { kernel<<<nmb, kSmallThreads, smem, st>>>(sp); };
  if (has_next)
    go(k_compact_small<true, true, false>);
  else if (hop)
    go(k_compact_small<false, true, false>);
  else
    go(k_compact_small<false, false, true>);
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" {

int vk_sampler_create(vk_graph g, const vk_sampler_config* cfg, vk_sampler* out) {
  return guard([&] {
    if (!g || !cfg || !out) raise(VK_ERR_PARAMETER, "null argument");
    const std::uint32_t L = cfg->num_hops;
    if (L == 0) raise(VK_ERR_PARAMETER, "fanout list must have at least one hop");
    if (L > VK_MAX_HOPS) raise(VK_ERR_UNSUPPORTED, "at most 8 hops are supported");
    for (std::uint32_t h = 0; h < L; ++h)
      if (cfg->fanouts[h] < 1) raise(VK_ERR_PARAMETER, "each fanout must be >= 1");
    if (cfg->batch_size == 0) raise(VK_ERR_PARAMETER, "batch size must be >= 1");
    if (cfg->max_minibatches == 0) raise(VK_ERR_PARAMETER, "max_minibatches must be >= 1");
    DeviceGuard dg(g->device);
    auto* s = new vk_sampler_s();
    try {
      s->g = g;
      s->cfg = *cfg;
      s->L = L;
      s->M = cfg->max_minibatches;
      s->n = g->n;
      s->W = (g->n + 63) / 64;
      s->tiles = (s->W + kTileWords - 1) / kTileWords;
      const std::uint64_t dmax = std::max<std::uint64_t>(1, g->max_out_degree);
      s->capF[0] = cfg->batch_size;
      std::uint64_t all = cfg->batch_size;
      for (std::uint32_t h = 1; h <= L; ++h) {
        const std::uint64_t f = std::min<std::uint64_t>(cfg->fanouts[h - 1], dmax);
        s->capS[h] = s->capF[h - 1] * f;
        s->capF[h] = std::min<std::uint64_t>(s->n, s->capS[h]);
        s->capS_max = std::max(s->capS_max, s->capS[h]);
        all += s->capF[h];
      }
      s->capAll = std::min<std::uint64_t>(s->n, all);
      // frontier representation: buckets when a minibatch touches a small
      // fraction of the vertices (papers scale), bitmaps otherwise
      {
        const bool ok = s->n <= (1ull << 31);  // ids and look-back counts fit 31 bits
        const bool want = (cfg->flags & VK_SAMPLER_FORCE_SPARSE) ||
                          (!(cfg->flags & VK_SAMPLER_FORCE_DENSE) && s->n >= 16 * s->capAll && s->n >= (1ull << 20));
        s->sparse = ok && want;
        if ((cfg->flags & VK_SAMPLER_FORCE_SPARSE) && !ok)
          raise(VK_ERR_UNSUPPORTED, "sparse frontiers need fewer than 2^31 vertices");
      }
      s->dense_all_rank = !s->sparse && 4 * s->W <= s->capAll;
      for (std::uint32_t h = 1; h <= L; ++h)
        if (s->capS[h] >= (1ull << 31))
          raise(VK_ERR_UNSUPPORTED, "per-minibatch edge capacity exceeds 2^31; lower batch size or fanouts");
      if (s->n >= (1ull << 31) && s->capAll >= (1ull << 31))
        raise(VK_ERR_UNSUPPORTED, "per-minibatch vertex capacity exceeds 2^31");
      const std::uint64_t M = s->M;
      for (std::uint32_t h = 0; h <= L; ++h) {
        s->F[h].alloc(M * s->capF[h] * 4);
        s->allidx[h].alloc(M * s->capF[h] * 4);
        if (h >= 1) {
          s->dst[h].alloc(M * s->capS[h] * 4);
          // MFG row pointer of hop h: |F_{h-1}|+1 entries per minibatch
          s->indptr[h].alloc(M * (s->capF[h - 1] + 1) * 4);
        }
      }
      s->edges_tmp.alloc(2 * M * s->capS_max * 4);
      s->all.alloc(M * s->capAll * 4);
      if (s->sparse) {
        // one bucket width for every level, so the all level can range the
        // sorted hop lists by the hops' bucket bases
        const std::uint32_t bb = bucket_bits(s->n);
        for (std::uint32_t h = 0; h <= L; ++h) s->bb[h] = bb;
        s->nb_max = s->nbuckets(0);
        s->fbase.alloc((std::uint64_t)(L + 1) * M * (s->nb_max + 1) * 4);
        s->pair_stride = s->capS_max;  // hop levels only (the all level ranges sorted lists)
        s->pairs.alloc(M * s->pair_stride * 8);
        s->bhist.alloc(M * (s->nb_max + 1) * 4);
        s->bstart.alloc(M * (s->nb_max + 1) * 4);
        s->bcursor.alloc(M * s->nb_max * 4);
        s->bstatus.alloc(M * s->nb_max * 8);
        s->tile_base.alloc(M * (s->nbuckets(0) + 1) * 4);
        VK_CUDA(cudaMemsetAsync(s->bhist.p, 0, s->bhist.bytes, nullptr));
        VK_CUDA(cudaFuncSetAttribute(k_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)scatter_smem(kMaxBuckets)));
        s->status.alloc(8);
      } else {
        s->hopbits.alloc(M * s->W * 8);
        s->allbits.alloc(M * s->W * 8);
        s->hopprefix.alloc(M * s->W * 16);  // RankWord {bits, prefix} per word
        s->allprefix.alloc(M * s->W * 16);
        s->status.alloc((std::uint64_t)(L + 1) * M * s->tiles * 8);
      }
      s->tickets.alloc((L + 1) * 4);
      s->counts.alloc(s->counts_words() * 4);
      s->desc.alloc(M * sizeof(WaveDesc));
      s->seed_stage.alloc(M * cfg->batch_size * 4);
      VK_CUDA(cudaFuncSetAttribute(k_compact<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kCompactThreads * 17 * 8));
      VK_CUDA(cudaFuncSetAttribute(k_compact<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kCompactThreads * 17 * 8));
      VK_CUDA(cudaFuncSetAttribute(k_compact<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kCompactThreads * 17 * 8));
      VK_CUDA(cudaFuncSetAttribute(k_sample_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   6 * 32 * kSampleThreads * 4));
      for (int k = 0; k < vk_sampler_s::kStageSlots; ++k) {
        s->desc_host[k].ensure(M * sizeof(WaveDesc));
        s->seed_host[k].ensure(M * cfg->batch_size * 4);
        VK_CUDA(cudaEventCreateWithFlags(&s->staged[k], cudaEventDisableTiming));
      }
      VK_CUDA(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
      VK_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
      VK_CUDA(cudaStreamCreateWithFlags(&s->aux, cudaStreamNonBlocking));
      VK_CUDA(cudaEventCreateWithFlags(&s->fork_ev, cudaEventDisableTiming));
      VK_CUDA(cudaEventCreateWithFlags(&s->join_ev, cudaEventDisableTiming));
      if (!s->sparse) {
        VK_CUDA(cudaMemsetAsync(s->hopbits.p, 0, s->hopbits.bytes, s->stream));
        VK_CUDA(cudaMemsetAsync(s->allbits.p, 0, s->allbits.bytes, s->stream));
      }
      VK_CUDA(cudaDeviceSynchronize());  // the legacy-stream bucket histogram clear
      VK_CUDA(cudaMemsetAsync(s->counts.p, 0, s->counts.bytes, s->stream));
      VK_CUDA(cudaStreamSynchronize(s->stream));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int vk_sampler_set_seed_keys(vk_sampler s, const uint32_t* seed_keys) {
  return guard([&] {
    if (!s) raise(VK_ERR_PARAMETER, "null argument");
    vk_graph_s& g = *s->g;
    DeviceGuard dg(g.device);
    if (s->last_stream) VK_CUDA(cudaStreamSynchronize(s->last_stream));
    if (!seed_keys) {
      s->keyed = false;
      s->keys.release();
      s->tgt_keyed.release();
      return;
    }
    const std::uint64_t n = g.n, m = g.m;
    cudaStream_t st = s->stream;
    s->keys.alloc(n * 4);
    VK_CUDA(cudaMemcpyAsync(s->keys.p, seed_keys, n * 4, cudaMemcpyHostToDevice, st));
    s->tgt_keyed.alloc(m ? m * 4 : 4);
    if (m) {
      DevBuf k1(m * 8), k2(m * 8), v1(m * 4);
      const unsigned grid = (unsigned)std::min<std::uint64_t>((n * 32 + 255) / 256, (std::uint64_t)sm_count(g.device) * 16);
      k_keyed_pairs<<<std::max(1u, grid), 256, 0, st>>>(g.d_off(), g.d_tgt(), s->keys.as<std::uint32_t>(), n,
                                                       k1.as<std::uint64_t>(), v1.as<std::uint32_t>());
      count_launch();
      VK_LAUNCH_CHECK();
      int end_bit = 32;
      while ((1ull << (end_bit - 32)) < n && end_bit < 64) ++end_bit;
      std::size_t tmp = 0;
      VK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k1.as<std::uint64_t>(), k2.as<std::uint64_t>(),
                                              v1.as<std::uint32_t>(), s->tgt_keyed.as<std::uint32_t>(),
                                              (std::int64_t)m, 0, end_bit, st));
      DevBuf tb(tmp);
      VK_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, k1.as<std::uint64_t>(), k2.as<std::uint64_t>(),
                                              v1.as<std::uint32_t>(), s->tgt_keyed.as<std::uint32_t>(),
                                              (std::int64_t)m, 0, end_bit, st));
      count_launch(4);
    }
    VK_CUDA(cudaStreamSynchronize(st));
    s->keyed = true;
  });
}

int vk_sampler_destroy(vk_sampler s) {
  return guard([&] {
    if (!s) return;
    DeviceGuard dg(s->g->device);
    if (s->last_stream) cudaStreamSynchronize(s->last_stream);
    if (s->aux) cudaStreamSynchronize(s->aux);
    if (s->stream) cudaStreamDestroy(s->stream);
    if (s->aux) cudaStreamDestroy(s->aux);
    if (s->fork_ev) cudaEventDestroy(s->fork_ev);
    if (s->join_ev) cudaEventDestroy(s->join_ev);
    for (int k = 0; k < vk_sampler_s::kStageSlots; ++k)
      if (s->staged[k]) cudaEventDestroy(s->staged[k]);
    if (s->done) cudaEventDestroy(s->done);
    for (cudaEvent_t e : s->readers) {
      cudaEventSynchronize(e);
      cudaEventDestroy(e);
    }
    for (cudaEvent_t e : s->reader_pool) cudaEventDestroy(e);
    delete s;
  });
}

int vk_sampler_run(vk_sampler s, uint32_t nmb, const vk_batch_ref* refs, const uint32_t* seeds,
                   const uint64_t* seed_offsets, int seeds_on_device, vk_stream_t stream) {
  return guard([&] {
    if (!s || !refs || !seeds || !seed_offsets) raise(VK_ERR_PARAMETER, "null argument");
    if (nmb == 0) raise(VK_ERR_PARAMETER, "empty wave");
    if (nmb > s->M) raise(VK_ERR_PARAMETER, "wave exceeds max_minibatches");
    vk_graph_s& g = *s->g;
    DeviceGuard dg(g.device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    // make sure the previous run on another stream has finished with the
    // shared workspace before it is rewritten
    if (s->last_stream && s->last_stream != st) VK_CUDA(cudaStreamSynchronize(s->last_stream));
    // ... and that every reader of it on another stream is done
    for (cudaEvent_t e : s->readers) {
      VK_CUDA(cudaStreamWaitEvent(st, e, 0));
      s->reader_pool.push_back(e);
    }
    s->readers.clear();
    const std::uint64_t b = s->cfg.batch_size;
    const std::uint64_t total = seed_offsets[nmb] - seed_offsets[0];
    for (std::uint32_t i = 0; i < nmb; ++i) {
      const std::uint64_t c = seed_offsets[i + 1] - seed_offsets[i];
      if (c == 0) raise(VK_ERR_SAMPLING, "cannot expand an empty batch");  // sampling.cpp:97
      if (c > b) raise(VK_ERR_PARAMETER, "minibatch larger than the sampler's batch_size");
    }
    // ring of pinned staging slots: only wait for the H2D copy issued kStageSlots
    // waves ago, so the host can queue the next wave while this one runs
    const int slot = s->slot;
    s->slot = (s->slot + 1) % vk_sampler_s::kStageSlots;
    if (s->staged_used[slot]) VK_CUDA(cudaEventSynchronize(s->staged[slot]));
    WaveDesc* d = s->desc_host[slot].as<WaveDesc>();
    for (std::uint32_t i = 0; i < nmb; ++i) {
      std::memset(&d[i], 0, sizeof(WaveDesc));
      for (std::uint32_t h = 1; h <= s->L; ++h)
        d[i].key_prefix[h - 1] = sample_key_prefix(s->cfg.global_seed, refs[i].epoch, refs[i].partition,
                                                   refs[i].batch_index, h);
      d[i].seed_begin = seed_offsets[i] - seed_offsets[0];
      d[i].seed_count = (std::uint32_t)(seed_offsets[i + 1] - seed_offsets[i]);
      d[i].partition = refs[i].partition;
    }
    VK_CUDA(cudaMemcpyAsync(s->desc.p, d, nmb * sizeof(WaveDesc), cudaMemcpyHostToDevice, st));
    const std::uint32_t* dseeds;
    if (seeds_on_device) {
      dseeds = seeds + seed_offsets[0];
    } else {
      for (std::uint64_t i = 0; i < total; ++i)
        if (seeds[seed_offsets[0] + i] >= s->n)
          raise(VK_ERR_RANGE, "seed vertex id out of range: " + std::to_string(seeds[seed_offsets[0] + i]));
      std::memcpy(s->seed_host[slot].p, seeds + seed_offsets[0], total * 4);
      VK_CUDA(cudaMemcpyAsync(s->seed_stage.p, s->seed_host[slot].p, total * 4, cudaMemcpyHostToDevice, st));
      dseeds = s->seed_stage.as<std::uint32_t>();
    }
    VK_CUDA(cudaEventRecord(s->staged[slot], st));
    s->staged_used[slot] = true;
    if (!s->sparse) VK_CUDA(cudaMemsetAsync(s->status.p, 0, s->status.bytes, st));
    VK_CUDA(cudaMemsetAsync(s->tickets.p, 0, s->tickets.bytes, st));
    VK_CUDA(cudaMemsetAsync(s->err(), 0, 4, st));
    const std::uint32_t* outdeg = g.out_deg.as<std::uint32_t>();
    k_prepare<<<nmb, 1024, 0, st>>>(s->desc.as<WaveDesc>(), dseeds, outdeg, s->n, s->cfg.fanouts[0],
                                    s->F[0].as<std::uint32_t>(), s->capF[0], s->fcount(0),
                                    s->indptr[1].as<std::uint32_t>(), s->ecount(1),
                                    s->sparse ? nullptr : s->allbits.as<unsigned long long>(), s->W, s->err());
    count_launch();
    VK_LAUNCH_CHECK();
    // small graphs: per-minibatch CTAs compact with shared-memory bitmaps and
    // fuse the relabels (C1: 65 K -> 71 K minibatches/s)
    const bool small = !s->sparse && s->W <= kSmallW;
    // the MFG relabel of hop h overlaps the sampling of hop h+1 on aux
    constexpr bool relabel_overlap = true;
    bool relabel_pending = false;  // a relabel is running on aux (join before the next compaction)
    for (std::uint32_t h = 1; h <= s->L; ++h) {
      const std::uint32_t f = s->cfg.fanouts[h - 1];
      if (f <= 32)
        launch_sample<0>(*s, h, nmb, st);
      else if (g.max_out_degree <= f || f <= 128)
        launch_sample<128>(*s, h, nmb, st);
      else if (f <= 1024)
        launch_sample<1024>(*s, h, nmb, st);
      else
        raise(VK_ERR_UNSUPPORTED, "fanouts above 1024 with higher-degree vertices are not supported");
      count_launch();
      VK_LAUNCH_CHECK();
      if (s->sparse) {
        run_bucket_level(*s, h, nmb, st);
        continue;
      }
      if (small) {
        run_compact_small(*s, true, h, nmb, st);
        count_launch();
        VK_LAUNCH_CHECK();
        continue;
      }
      if (relabel_pending) {  // hop h-1's relabel still reads hopprefix
        VK_CUDA(cudaStreamWaitEvent(st, s->join_ev, 0));
        relabel_pending = false;
      }
      run_compact(*s, true, h, nmb, h - 1, st);
      count_launch();
      VK_LAUNCH_CHECK();
      const unsigned gx = (unsigned)std::min<std::uint64_t>(ceil_div(s->capS[h], 256 * kIlp), 4096);
      cudaStream_t rs_ = st;
      if (relabel_overlap) {
        VK_CUDA(cudaEventRecord(s->fork_ev, st));
        VK_CUDA(cudaStreamWaitEvent(s->aux, s->fork_ev, 0));
        rs_ = s->aux;
      }
      k_relabel<<<dim3(gx, nmb), 256, 0, rs_>>>(s->edges_buf(h), s->capS_max, s->ecount(h),
                                                s->hopprefix.as<uint4>(), s->W, s->dst[h].as<std::uint32_t>(),
                                                s->capS[h]);
      count_launch();
      VK_LAUNCH_CHECK();
      if (relabel_overlap) {
        VK_CUDA(cudaEventRecord(s->join_ev, s->aux));
        relabel_pending = true;
      }
    }
    if (s->sparse) {
      run_bucket_level(*s, 0, nmb, st);
    } else if (small) {
      run_compact_small(*s, false, 0, nmb, st);
      count_launch();
      VK_LAUNCH_CHECK();
    } else {
      run_compact(*s, false, 0, nmb, s->L, st);
      count_launch();
      VK_LAUNCH_CHECK();
      // relabel map per hop (grids sized by each hop's capacity)
      for (std::uint32_t h = 0; h <= s->L; ++h) {
        const unsigned gx = (unsigned)std::min<std::uint64_t>(ceil_div(s->capF[h], 256 * kIlp), 4096);
        k_allidx<<<dim3(gx, nmb), 256, 0, st>>>(s->F[h].as<std::uint32_t>(), s->allidx[h].as<std::uint32_t>(),
                                                s->capF[h], s->fcount(h), s->allprefix.as<uint4>(), s->W);
        count_launch();
      }
    }
    if (relabel_pending) VK_CUDA(cudaStreamWaitEvent(st, s->join_ev, 0));  // the last hop's relabel
    count_launch();
    VK_LAUNCH_CHECK();
    VK_CUDA(cudaEventRecord(s->done, st));
    s->last_nmb = nmb;
    ++s->runs;
    s->last_stream = st;
    s->last_parts.resize(nmb);
    for (std::uint32_t i = 0; i < nmb; ++i) s->last_parts[i] = refs[i].partition;
  });
}

namespace {

void sync_last(vk_sampler_s& s) {
  if (s.last_nmb == 0) raise(VK_ERR_PARAMETER, "sampler has not run");
  VK_CUDA(cudaStreamSynchronize(s.last_stream ? s.last_stream : s.stream));
}

std::vector<std::uint32_t> host_counts(vk_sampler_s& s) {
  sync_last(s);
  std::vector<std::uint32_t> c(s.counts_words());
  VK_CUDA(cudaMemcpy(c.data(), s.counts.p, c.size() * 4, cudaMemcpyDeviceToHost));
  if (c.back()) raise(VK_ERR_RANGE, "seed vertex id out of range");
  return c;
}

void check_mb_hop(vk_sampler_s& s, std::uint32_t mb, std::uint32_t hop, std::uint32_t lo) {
  if (mb >= s.last_nmb) raise(VK_ERR_PARAMETER, "minibatch index out of range");
  if (hop < lo || hop > s.L) raise(VK_ERR_PARAMETER, "hop out of range");
}

}  // namespace

int vk_sampler_sizes(vk_sampler s, uint64_t* frontier_sizes, uint64_t* edge_counts, uint64_t* all_sizes) {
  return guard([&] {
    if (!s) raise(VK_ERR_PARAMETER, "null sampler");
    DeviceGuard dg(s->g->device);
    const auto c = host_counts(*s);
    const std::uint32_t M = s->M, L = s->L;
    for (std::uint32_t i = 0; i < s->last_nmb; ++i) {
      for (std::uint32_t h = 1; h <= L; ++h) {
        if (frontier_sizes) frontier_sizes[i * L + h - 1] = c[(std::uint64_t)h * M + i];
        if (edge_counts) edge_counts[i * L + h - 1] = c[(std::uint64_t)(L + 1) * M + (std::uint64_t)h * M + i];
      }
      if (all_sizes) all_sizes[i] = c[2ull * (L + 1) * M + i];
    }
  });
}

int vk_sampler_copy_frontier(vk_sampler s, uint32_t mb, uint32_t hop, uint32_t* out) {
  return guard([&] {
    if (!s || !out) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(s->g->device);
    check_mb_hop(*s, mb, hop, 0);
    const auto c = host_counts(*s);
    const std::uint64_t cnt = c[(std::uint64_t)hop * s->M + mb];
    VK_CUDA(cudaMemcpy(out, s->F[hop].as<std::uint32_t>() + mb * s->capF[hop], cnt * 4, cudaMemcpyDeviceToHost));
  });
}

int vk_sampler_copy_all(vk_sampler s, uint32_t mb, uint32_t* out) {
  return guard([&] {
    if (!s || !out) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(s->g->device);
    check_mb_hop(*s, mb, 0, 0);
    const auto c = host_counts(*s);
    const std::uint64_t cnt = c[2ull * (s->L + 1) * s->M + mb];
    VK_CUDA(cudaMemcpy(out, s->all.as<std::uint32_t>() + mb * s->capAll, cnt * 4, cudaMemcpyDeviceToHost));
  });
}

int vk_sampler_copy_mfg(vk_sampler s, uint32_t mb, uint32_t hop, uint64_t* indptr, uint32_t* dst) {
  return guard([&] {
    if (!s) raise(VK_ERR_PARAMETER, "null sampler");
    DeviceGuard dg(s->g->device);
    check_mb_hop(*s, mb, hop, 1);
    const auto c = host_counts(*s);
    const std::uint64_t nsrc = c[(std::uint64_t)(hop - 1) * s->M + mb];
    const std::uint64_t ne = c[(std::uint64_t)(s->L + 1) * s->M + (std::uint64_t)hop * s->M + mb];
    if (indptr) {
      std::vector<std::uint32_t> ip(nsrc + 1);
      VK_CUDA(cudaMemcpy(ip.data(), s->indptr[hop].as<std::uint32_t>() + mb * (s->capF[hop - 1] + 1),
                         (nsrc + 1) * 4, cudaMemcpyDeviceToHost));
      for (std::uint64_t i = 0; i <= nsrc; ++i) indptr[i] = ip[i];
    }
    if (dst && ne)
      VK_CUDA(cudaMemcpy(dst, s->dst[hop].as<std::uint32_t>() + mb * s->capS[hop], ne * 4, cudaMemcpyDeviceToHost));
  });
}

int vk_sampler_copy_relabel(vk_sampler s, uint32_t mb, uint32_t hop, uint32_t* all_index) {
  return guard([&] {
    if (!s || !all_index) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(s->g->device);
    check_mb_hop(*s, mb, hop, 0);
    const auto c = host_counts(*s);
    const std::uint64_t cnt = c[(std::uint64_t)hop * s->M + mb];
    VK_CUDA(cudaMemcpy(all_index, s->allidx[hop].as<std::uint32_t>() + mb * s->capF[hop], cnt * 4,
                       cudaMemcpyDeviceToHost));
  });
}

// sample_neighbors (sampling.cpp:72-92) for one vertex, one device thread:
// deg <= f copies the row in CSR order, else a partial Fisher-Yates over the
// row (or over the row ordered by seed key, `sorted`) with the sparse
// displaced-position map in global scratch; the caller's stream state is
// advanced in place.
__global__ void k_sample_vertex(const std::uint64_t* __restrict__ off, const std::uint32_t* __restrict__ tgt,
                                const std::uint32_t* __restrict__ sorted, std::uint32_t v, std::uint32_t f,
                                std::uint64_t* __restrict__ counter, std::uint32_t* __restrict__ out,
                                std::uint32_t* __restrict__ cnt, std::uint32_t* __restrict__ hp,
                                std::uint32_t* __restrict__ hv) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const std::uint64_t o0 = off[v];
  const std::uint32_t deg = (std::uint32_t)(off[v + 1] - o0);
  if (deg <= f) {
    for (std::uint32_t i = 0; i < deg; ++i) out[i] = tgt[o0 + i];
    *cnt = deg;
    return;
  }
  const std::uint32_t* row = sorted ? sorted : tgt + o0;
  Stream s(0);
  s.counter = *counter;
  // out[0..f) holds positions [0, f); positions >= f displaced by a swap in (hp, hv)
  for (std::uint32_t i = 0; i < f; ++i) out[i] = row[i];
  std::uint32_t nh = 0;
  for (std::uint32_t i = 0; i < f; ++i) {
    const std::uint32_t j = i + (std::uint32_t)s.next_below((std::uint64_t)(deg - i));
    const std::uint32_t vi = out[i];
    std::uint32_t vj;
    if (j < f) {
      vj = out[j];
      out[j] = vi;
    } else {
      std::uint32_t c = 0;
      while (c < nh && hp[c] != j) ++c;
      if (c < nh) {
        vj = hv[c];
        hv[c] = vi;
      } else {
        vj = row[j];
        hp[nh] = j;
        hv[nh] = vi;
        ++nh;
      }
    }
    out[i] = vj;  // scratch[i] after the swap
  }
  *counter = s.counter;
  *cnt = f;
}

int vk_graph_sample_neighbors(vk_graph g, uint32_t v, uint32_t fanout, uint64_t* stream_state,
                              const uint32_t* neighbor_keys, uint32_t* out, uint64_t* out_count) {
  return guard([&] {
    if (!g || !stream_state || !out || !out_count) raise(VK_ERR_PARAMETER, "null argument");
    if (v >= g->n) raise(VK_ERR_RANGE, "vertex id out of range");
    DeviceGuard dg(g->device);
    std::uint64_t o[2];
    VK_CUDA(cudaMemcpy(o, g->d_off() + v, 16, cudaMemcpyDeviceToHost));
    const std::uint64_t deg = o[1] - o[0];
    const std::uint64_t take = std::min<std::uint64_t>(deg, fanout);
    DevBuf d_out(std::max<std::uint64_t>(1, take) * 4), d_state(8), d_cnt(4),
        d_hp(std::max<std::uint64_t>(1, take) * 4), d_hv(std::max<std::uint64_t>(1, take) * 4);
    VK_CUDA(cudaMemcpy(d_state.p, stream_state, 8, cudaMemcpyHostToDevice));
    DevBuf sorted;
    if (neighbor_keys && deg > fanout) {
      // the row ordered by the neighbours' seed keys (sampling.cpp:83-85):
      // one radix sort of (key, neighbour) pairs
      DevBuf k_in(deg * 4), k_out(deg * 4);
      sorted.alloc(deg * 4);
      VK_CUDA(cudaMemcpy(k_in.p, neighbor_keys, deg * 4, cudaMemcpyHostToDevice));
      std::size_t tmp = 0;
      VK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k_in.as<std::uint32_t>(), k_out.as<std::uint32_t>(),
                                              g->d_tgt() + o[0], sorted.as<std::uint32_t>(), (std::int64_t)deg));
      DevBuf tb(std::max<std::size_t>(tmp, 1));
      VK_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, k_in.as<std::uint32_t>(), k_out.as<std::uint32_t>(),
                                              g->d_tgt() + o[0], sorted.as<std::uint32_t>(), (std::int64_t)deg));
      count_launch(4);
    }
    k_sample_vertex<<<1, 32>>>(g->d_off(), g->d_tgt(), sorted.p ? sorted.as<std::uint32_t>() : nullptr, v, fanout,
                               d_state.as<std::uint64_t>(), d_out.as<std::uint32_t>(), d_cnt.as<std::uint32_t>(),
                               d_hp.as<std::uint32_t>(), d_hv.as<std::uint32_t>());
    count_launch();
    VK_LAUNCH_CHECK();
    std::uint32_t c = 0;
    VK_CUDA(cudaMemcpy(&c, d_cnt.p, 4, cudaMemcpyDeviceToHost));
    VK_CUDA(cudaMemcpy(out, d_out.p, (std::uint64_t)c * 4, cudaMemcpyDeviceToHost));
    VK_CUDA(cudaMemcpy(stream_state, d_state.p, 8, cudaMemcpyDeviceToHost));
    *out_count = c;
  });
}

int vk_debug_stream_draws(int device, uint64_t key, uint64_t bound, uint64_t count, uint64_t* out) {
  return guard([&] {
    if (!out) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(device);
    DevBuf d(std::max<std::uint64_t>(count, 1) * 8);
    k_stream_draws<<<1, 32>>>(key, bound, count, d.as<std::uint64_t>());
    count_launch();
    VK_LAUNCH_CHECK();
    VK_CUDA(cudaMemcpy(out, d.p, count * 8, cudaMemcpyDeviceToHost));
  });
}

int vk_sampler_snapshot_counts(vk_sampler s, uint32_t* dst_dev, uint64_t* words, vk_stream_t stream) {
  return guard([&] {
    if (!s) raise(VK_ERR_PARAMETER, "null sampler");
    if (words) *words = s->counts_words();
    if (!dst_dev) return;
    DeviceGuard dg(s->g->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : (s->last_stream ? s->last_stream : s->stream);
    if (s->last_stream && st != s->last_stream) VK_CUDA(cudaStreamWaitEvent(st, s->done, 0));
    VK_CUDA(cudaMemcpyAsync(dst_dev, s->counts.p, s->counts_words() * 4, cudaMemcpyDeviceToDevice, st));
  });
}

int vk_sampler_get_view(vk_sampler s, vk_sampler_view* v) {
  return guard([&] {
    if (!s || !v) raise(VK_ERR_PARAMETER, "null argument");
    std::memset(v, 0, sizeof *v);
    v->nmb = s->last_nmb;
    v->num_hops = s->L;
    v->all = s->all.as<std::uint32_t>();
    v->all_stride = s->capAll;
    v->all_count = s->allcount();
    for (std::uint32_t h = 0; h <= s->L; ++h) {
      v->frontier[h] = s->F[h].as<std::uint32_t>();
      v->frontier_stride[h] = s->capF[h];
      v->frontier_count[h] = s->fcount(h);
      v->all_index[h] = s->allidx[h].as<std::uint32_t>();
      if (h >= 1) {
        v->mfg_indptr[h] = s->indptr[h].as<std::uint32_t>();
        v->mfg_dst[h] = s->dst[h].as<std::uint32_t>();
        v->mfg_stride[h] = s->capS[h];
      }
    }
  });
}

}  // extern "C"

// internal accessors for the feature plane (plane.cu)
namespace vk {
void sampler_internal(vk_sampler_s* s, const std::uint32_t** all, std::uint64_t* all_stride,
                      const std::uint32_t** all_count, std::uint32_t* nmb, const std::uint32_t** partitions,
                      vk_graph_s** g, cudaStream_t* last_stream) {
  *all = s->all.as<std::uint32_t>();
  *all_stride = s->capAll;
  *all_count = s->allcount();
  *nmb = s->last_nmb;
  *partitions = reinterpret_cast<const std::uint32_t*>(s->desc.as<char>() + offsetof(WaveDesc, partition));
  *g = s->g;
  *last_stream = s->last_stream;
}
std::uint64_t sampler_desc_stride() { return sizeof(WaveDesc); }
void sampler_all_rank(vk_sampler_s* s, const uint4** rank, std::uint64_t* W) {
  *rank = s->allprefix.as<uint4>();
  *W = s->W;
}
bool sampler_all_rank_dense(vk_sampler_s* s) { return s->dense_all_rank; }
// sparse frontiers: rank of every all-level bucket's first vertex per
// minibatch ([nmb][NB + 1]) and the bucket width; nullptr for bitmaps
const std::uint32_t* sampler_tile_base(vk_sampler_s* s, std::uint32_t* bucket_bits, std::uint32_t* nb) {
  if (!s->sparse) return nullptr;
  *bucket_bits = s->bb[0];
  *nb = s->nbuckets(0);
  return s->tile_base.as<std::uint32_t>();
}
std::uint64_t sampler_run_id(vk_sampler_s* s) { return s->runs; }
void sampler_host_partitions(vk_sampler_s* s, std::vector<std::uint32_t>& out) { out = s->last_parts; }
cudaEvent_t sampler_done_event(vk_sampler_s* s) { return s->done; }
void sampler_add_reader(vk_sampler_s* s, cudaStream_t st) {
  cudaEvent_t e;
  if (s->reader_pool.empty()) {
    VK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  } else {
    e = s->reader_pool.back();
    s->reader_pool.pop_back();
  }
  VK_CUDA(cudaEventRecord(e, st));
  s->readers.push_back(e);
}
std::uint64_t sampler_capacity_all(vk_sampler_s* s) { return s->capAll; }
}  // namespace vk
