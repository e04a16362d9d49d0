// Sparse frontiers (papers-scale graphs): per-minibatch dedup + relabel by
// vertex-range buckets instead of an n-bit global bitmap.
//
// When a frontier holds a small fraction of the n vertices (C4: |F_h| <= 0.7%
// of 111 M), scanning, clearing and ranking n/64 bitmap words per minibatch
// per level -- and one random global RED per sampled edge -- cost ~25x the
// algorithmic bytes (r02 launch list). Here a level's items (the hop's drawn
// ids in MFG order, or for the all level the lists F_0..F_L) are
//   1. counted per (minibatch, bucket of 2^bb consecutive ids)   k_bucket_hist
//   2. scanned to bucket offsets                                  k_bucket_scan
//   3. scattered as (id, tag) pairs into bucket order             k_bucket_scatter
//   4. deduplicated per bucket in a shared-memory bitmap, ranked with a
//      block scan + decoupled look-back across the minibatch's buckets, and
//      emitted: the sorted distinct list (sort + unique of sampling.cpp:
//      115-116 and 121-126), the next hop's MFG row pointers, and every
//      pair's rank (MFG dst / all_vertices index)                 k_bucket_dedup
// Items and pairs stream through HBM once or twice; the bitmap work stays in
// shared memory. Results are identical to the dense (bitmap) path.
#pragma once

namespace vk {
namespace {

constexpr int kBktThreads = 256;
constexpr std::uint32_t kChunkItems = 4096;  // items per (chunk, minibatch) CTA of hist / scatter
constexpr std::uint32_t kMaxBuckets = 8192;  // per minibatch (shared histogram of hist / scatter)
constexpr std::uint32_t kTagLevelShift = 28;  // all level: tag = level << 28 | index in F_level

struct BucketParams {
  // hop level: items ids[mb * ids_stride + i], i < count[mb], tag = i
  const std::uint32_t* ids;
  std::uint64_t ids_stride;
  const std::uint32_t* count;
  // all level (ids == nullptr): F_0..F_L, tag = level << 28 | index
  std::uint32_t L;
  const std::uint32_t* F[VK_MAX_HOPS + 1];
  std::uint64_t capF[VK_MAX_HOPS + 1];
  const std::uint32_t* fcount[VK_MAX_HOPS + 1];
  std::uint32_t bb, NB;     // bucket = id >> bb, NB buckets per minibatch
  std::uint32_t* hist;      // [M][NB + 1], zero between levels
  std::uint32_t* bstart;    // [M][NB + 1] pair offset of every bucket
  std::uint32_t* cursor;    // [M][NB]
  uint2* pairs;             // [M][pair_stride] {id, tag}
  std::uint64_t pair_stride;
  unsigned long long* status;  // [M][NB] look-back of the dedup (reset by the scan)
};

// The i-th item of minibatch mb (all level: `pre` = level starts).
__device__ __forceinline__ uint2 bucket_item(const BucketParams& p, std::uint32_t mb, std::uint32_t i,
                                             const std::uint32_t* pre) {
  if (p.ids) return make_uint2(__ldg(p.ids + mb * p.ids_stride + i), i);
  std::uint32_t h = 0;
  while (i >= pre[h + 1]) ++h;
  const std::uint32_t idx = i - pre[h];
  return make_uint2(__ldg(p.F[h] + mb * p.capF[h] + idx), (h << kTagLevelShift) | idx);
}

// Item count of minibatch mb; all level: level starts into pre[0..L+1].
__device__ __forceinline__ std::uint32_t bucket_items(const BucketParams& p, std::uint32_t mb, std::uint32_t* pre) {
  if (p.ids) return p.count[mb];
  if (threadIdx.x == 0) {
    std::uint32_t a = 0;
    for (std::uint32_t h = 0; h <= p.L; ++h) {
      pre[h] = a;
      a += p.fcount[h][mb];
    }
    pre[p.L + 1] = a;
  }
  __syncthreads();
  return pre[p.L + 1];
}

// 1. per-bucket item counts; shared histogram per (chunk, minibatch) CTA
__global__ void __launch_bounds__(kBktThreads) k_bucket_hist(BucketParams p) {
  extern __shared__ std::uint32_t s_hist[];
  __shared__ std::uint32_t s_pre[VK_MAX_HOPS + 2];
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t total = bucket_items(p, mb, s_pre);
  const std::uint32_t c0 = blockIdx.x * kChunkItems;
  if (c0 >= total) return;
  const std::uint32_t c1 = min(total, c0 + kChunkItems);
  for (std::uint32_t b = threadIdx.x; b < p.NB; b += kBktThreads) s_hist[b] = 0;
  __syncthreads();
  for (std::uint32_t i = c0 + threadIdx.x; i < c1; i += kBktThreads)
    atomicAdd(&s_hist[bucket_item(p, mb, i, s_pre).x >> p.bb], 1u);
  __syncthreads();
  std::uint32_t* hist = p.hist + (std::uint64_t)mb * (p.NB + 1);
  for (std::uint32_t b = threadIdx.x; b < p.NB; b += kBktThreads)
    if (s_hist[b]) atomicAdd(hist + b, s_hist[b]);
}

// 2. bucket offsets (exclusive scan), cursors, look-back reset; the
// histogram is cleared for the next level. One CTA per minibatch.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_bucket_scan(BucketParams p) {
  __shared__ unsigned long long s_sm[kScanThreads / 32];
  const std::uint32_t mb = blockIdx.x;
  const std::uint32_t NB = p.NB;
  std::uint32_t* hist = p.hist + (std::uint64_t)mb * (NB + 1);
  std::uint32_t* bs = p.bstart + (std::uint64_t)mb * (NB + 1);
  std::uint32_t* cur = p.cursor + (std::uint64_t)mb * NB;
  unsigned long long* st = p.status + (std::uint64_t)mb * NB;
  const std::uint32_t per = (NB + kScanThreads - 1) / kScanThreads;
  const std::uint32_t b0 = min(NB, threadIdx.x * per), b1 = min(NB, b0 + per);
  unsigned long long mine = 0;
  for (std::uint32_t b = b0; b < b1; ++b) mine += hist[b];
  unsigned long long total;
  unsigned long long run = block_inclusive_scan<kScanThreads>(mine, s_sm, &total) - mine;
  for (std::uint32_t b = b0; b < b1; ++b) {
    const std::uint32_t c = hist[b];
    bs[b] = (std::uint32_t)run;
    cur[b] = (std::uint32_t)run;
    hist[b] = 0;
    st[b] = 0ull;
    run += c;
  }
  if (threadIdx.x == 0) bs[NB] = (std::uint32_t)total;
}

// 3. (id, tag) pairs into bucket order: the CTA reserves one range per
// bucket it touches (one global atomic per bucket), then places its items
// with shared cursors. Order inside a bucket is irrelevant (set semantics).
__global__ void __launch_bounds__(kBktThreads) k_bucket_scatter(BucketParams p) {
  extern __shared__ std::uint32_t s_dyn[];
  std::uint32_t* s_cnt = s_dyn;          // [NB]
  std::uint32_t* s_base = s_dyn + p.NB;  // [NB]
  __shared__ std::uint32_t s_pre[VK_MAX_HOPS + 2];
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t total = bucket_items(p, mb, s_pre);
  const std::uint32_t c0 = blockIdx.x * kChunkItems;
  if (c0 >= total) return;
  const std::uint32_t c1 = min(total, c0 + kChunkItems);
  for (std::uint32_t b = threadIdx.x; b < p.NB; b += kBktThreads) s_cnt[b] = 0;
  __syncthreads();
  for (std::uint32_t i = c0 + threadIdx.x; i < c1; i += kBktThreads)
    atomicAdd(&s_cnt[bucket_item(p, mb, i, s_pre).x >> p.bb], 1u);
  __syncthreads();
  std::uint32_t* cur = p.cursor + (std::uint64_t)mb * p.NB;
  for (std::uint32_t b = threadIdx.x; b < p.NB; b += kBktThreads) {
    const std::uint32_t c = s_cnt[b];
    if (c) s_base[b] = atomicAdd(cur + b, c);
    s_cnt[b] = 0;
  }
  __syncthreads();
  uint2* out = p.pairs + mb * p.pair_stride;
  for (std::uint32_t i = c0 + threadIdx.x; i < c1; i += kBktThreads) {
    const uint2 it = bucket_item(p, mb, i, s_pre);
    const std::uint32_t b = it.x >> p.bb;
    out[s_base[b] + atomicAdd(&s_cnt[b], 1u)] = it;
  }
}

struct DedupParams {
  BucketParams bp;
  unsigned* ticket;
  std::uint32_t nmb;
  std::uint32_t* list;  // F_h or all_vertices [M][cap_list]
  std::uint64_t cap_list;
  std::uint32_t* count;  // |F_h| or |all| [M]
  // hop level: dst[mb * dst_stride + tag] = rank (MFG relabel)
  std::uint32_t* dst;
  std::uint64_t dst_stride;
  // all level: allidx[h][mb * capF[h] + index] = rank; tile_base[mb][b] =
  // rank of bucket b's first vertex (the gather's vertex tiles)
  std::uint32_t* allidx[VK_MAX_HOPS + 1];
  std::uint32_t* tile_base;  // [M][NB + 1]
  // next hop's MFG row pointers over the list (HAS_NEXT)
  const std::uint32_t* outdeg;
  std::uint32_t f_next;
  std::uint32_t* indptr_next;  // [M][cap_list + 1]
  std::uint32_t* ecount_next;  // [M]
};

// 4. one CTA per (minibatch, bucket); tickets hand out buckets in ascending
// order per minibatch (minibatch fastest) so every look-back predecessor is
// already running. WPT = bitmap words per thread (bucket = 256*WPT*64 ids).
template <bool ALL, bool HAS_NEXT, int WPT>
__global__ void __launch_bounds__(kBktThreads) k_bucket_dedup(DedupParams p) {
  constexpr std::uint32_t BW = kBktThreads * WPT;  // words per bucket
  extern __shared__ unsigned long long s_bits[];   // [BW] bits, then u32 [BW] word ranks
  std::uint32_t* s_rank = reinterpret_cast<std::uint32_t*>(s_bits + BW);
  __shared__ unsigned s_ticket;
  __shared__ unsigned long long s_sm[kBktThreads / 32];
  __shared__ unsigned long long s_excl;
  const BucketParams& bp = p.bp;
  if (threadIdx.x == 0) s_ticket = atomicAdd(p.ticket, 1u);
  __syncthreads();
  const std::uint32_t mb = s_ticket % p.nmb;
  const std::uint32_t b = s_ticket / p.nmb;
  if (b >= bp.NB) return;
  const std::uint32_t NB = bp.NB;
  const std::uint32_t* bs = bp.bstart + (std::uint64_t)mb * (NB + 1);
  const std::uint32_t s = bs[b], e = bs[b + 1];
  unsigned long long* status = bp.status + (std::uint64_t)mb * NB;
  const bool last = b + 1 == NB;
  if (s == e && !ALL && !last) {  // empty bucket: an empty aggregate for the successors
    if (threadIdx.x == 0) publish_aggregate(status, b, 0ull);
    return;
  }
  const uint2* pairs = bp.pairs + mb * bp.pair_stride;
  const std::uint32_t vbase = b << bp.bb;
  for (std::uint32_t w = threadIdx.x; w < BW; w += kBktThreads) s_bits[w] = 0ull;
  __syncthreads();
  unsigned* bits32 = reinterpret_cast<unsigned*>(s_bits);
  for (std::uint32_t i = s + threadIdx.x; i < e; i += kBktThreads) {
    const std::uint32_t v = pairs[i].x - vbase;
    atomicOr(bits32 + (v >> 5), 1u << (v & 31));
  }
  __syncthreads();
  // this thread's WPT consecutive words: distinct count and capped degrees
  const std::uint32_t w0 = threadIdx.x * WPT;
  unsigned long long wd[WPT];
  unsigned long long vc = 0, dc = 0;
#pragma unroll
  for (int k = 0; k < WPT; ++k) {
    wd[k] = s_bits[w0 + k];
    vc += __popcll(wd[k]);
    if (HAS_NEXT && wd[k]) dc += capped_degree_sum(wd[k], (vbase >> 6) + w0 + k, p.outdeg, p.f_next);
  }
  const unsigned long long mine = pack_vd(vc, dc);
  unsigned long long total;
  const unsigned long long lex = block_inclusive_scan<kBktThreads>(mine, s_sm, &total) - mine;
  if (threadIdx.x == 0) publish_aggregate(status, b, total);
  if (threadIdx.x < 32) {
    const unsigned long long ex = lookback_resolve(status, b, total);
    if (threadIdx.x == 0) s_excl = ex;
  }
  __syncthreads();
  const unsigned long long base = s_excl;
  std::uint32_t gv = (std::uint32_t)(unpack_v(base) + unpack_v(lex));
  std::uint32_t gd = (std::uint32_t)(unpack_d(base) + unpack_d(lex));
  std::uint32_t* list = p.list + mb * p.cap_list;
  std::uint32_t* ipn = HAS_NEXT ? p.indptr_next + mb * (p.cap_list + 1) : nullptr;
#pragma unroll
  for (int k = 0; k < WPT; ++k) {
    s_rank[w0 + k] = gv;
    unsigned long long x = wd[k];
    const std::uint32_t wv = vbase + (w0 + k) * 64;
    while (x) {
      const int bit = __ffsll(x) - 1;
      x &= x - 1;
      const std::uint32_t v = wv + bit;
      list[gv] = v;
      if (HAS_NEXT) {
        ipn[gv] = gd;
        gd += min(p.f_next, __ldg(p.outdeg + v));
      }
      ++gv;
    }
  }
  if (ALL && threadIdx.x == 0) p.tile_base[mb * (NB + 1) + b] = (std::uint32_t)unpack_v(base);
  if (last && threadIdx.x == kBktThreads - 1) {
    const unsigned long long all = base + total;
    const std::uint32_t tv = (std::uint32_t)unpack_v(all), td = (std::uint32_t)unpack_d(all);
    p.count[mb] = tv;
    if (HAS_NEXT) {
      ipn[tv] = td;
      p.ecount_next[mb] = td;
    }
    if (ALL) p.tile_base[mb * (NB + 1) + NB] = tv;
  }
  __syncthreads();
  // every pair's rank: MFG dst (hop) or all_vertices index (all level)
  for (std::uint32_t i = s + threadIdx.x; i < e; i += kBktThreads) {
    const uint2 pr = pairs[i];
    const std::uint32_t v = pr.x - vbase, w = v >> 6;
    const std::uint32_t r = s_rank[w] + (std::uint32_t)__popcll(s_bits[w] & ((1ull << (v & 63)) - 1ull));
    if (ALL) {
      const std::uint32_t h = pr.y >> kTagLevelShift, idx = pr.y & ((1u << kTagLevelShift) - 1u);
      p.allidx[h][mb * bp.capF[h] + idx] = r;
    } else {
      p.dst[mb * p.dst_stride + pr.y] = r;
    }
  }
}

}  // namespace
}  // namespace vk
