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
constexpr std::uint32_t kHistItems = 16384;    // items per (chunk, minibatch) CTA of the histogram
constexpr std::uint32_t kScatterItems = 4096;  // ... of the scatter (16 per thread, held in registers)
constexpr std::uint32_t kMaxBuckets = 8192;  // per minibatch (shared histogram of hist / scatter)
constexpr std::uint32_t kItemBatch = 8;  // item loads in flight per thread (hist)

struct BucketParams {
  // hop level: items ids[mb * ids_stride + i], i < count[mb], tag = i (MFG position)
  const std::uint32_t* ids;
  std::uint64_t ids_stride;
  const std::uint32_t* count;
  // all level: the sorted lists F_1..F_L and the batch F_0 (k_bucket_dedup_all)
  std::uint32_t L;
  const std::uint32_t* F[VK_MAX_HOPS + 1];
  std::uint64_t capF[VK_MAX_HOPS + 1];
  const std::uint32_t* fcount[VK_MAX_HOPS + 1];
  std::uint32_t bb, NB;     // bucket = id >> bb, NB buckets per minibatch
  std::uint32_t* hist;      // [M][NB + 1], zero between levels
  std::uint32_t* bstart;    // [M][NB + 1] pair offset of every bucket
  std::uint32_t* cursor;    // [M][NB]
  uint2* pairs;             // [M][pair_stride] {id, MFG position}
  std::uint64_t pair_stride;
  unsigned long long* status;  // [M][NB] look-back of the dedup (reset by the scan)
};

// 1. per-bucket item counts; shared histogram per (chunk, minibatch) CTA
__global__ void __launch_bounds__(kBktThreads) k_bucket_hist(BucketParams p) {
  extern __shared__ std::uint32_t s_hist[];
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t total = p.count[mb];
  const std::uint32_t c0 = blockIdx.x * kHistItems;
  if (c0 >= total) return;
  const std::uint32_t c1 = min(total, c0 + kHistItems);
  const std::uint32_t* ids = p.ids + mb * p.ids_stride;
  for (std::uint32_t b = threadIdx.x; b < p.NB; b += kBktThreads) s_hist[b] = 0;
  __syncthreads();
  for (std::uint32_t i0 = c0 + threadIdx.x; i0 < c1; i0 += kItemBatch * kBktThreads) {
    std::uint32_t v[kItemBatch];  // loads in flight before their uses
#pragma unroll
    for (std::uint32_t k = 0; k < kItemBatch; ++k) {
      const std::uint32_t i = i0 + k * kBktThreads;
      v[k] = i < c1 ? __ldg(ids + i) : 0xffffffffu;
    }
#pragma unroll
    for (std::uint32_t k = 0; k < kItemBatch; ++k)
      if (v[k] != 0xffffffffu) atomicAdd(&s_hist[v[k] >> p.bb], 1u);
  }
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

// 3. (id, MFG position) pairs into bucket order: the CTA's kScatterItems
// items stay in registers with their rank inside their bucket (one shared
// atomic each); a block scan of the bucket counts sorts them by bucket in
// shared memory, the CTA reserves one range per bucket it touches (one global
// atomic per bucket), and the sorted pairs are written out so consecutive
// threads store consecutive addresses of a bucket's range (coalesced runs
// instead of one scattered 8-byte store per item). Order inside a bucket is
// irrelevant (set semantics).
constexpr std::size_t scatter_smem(std::uint32_t NB) {
  return ((std::size_t)3 * NB + 1) / 2 * 8 + (std::size_t)kScatterItems * 8;
}
__global__ void __launch_bounds__(kBktThreads) k_bucket_scatter(BucketParams p) {
  constexpr std::uint32_t kPer = kScatterItems / kBktThreads;
  extern __shared__ unsigned long long s_dyn8[];
  __shared__ unsigned long long s_sm[kBktThreads / 32];
  const std::uint32_t NB = p.NB;
  std::uint32_t* s_cnt = reinterpret_cast<std::uint32_t*>(s_dyn8);  // [NB]
  std::uint32_t* s_base = s_cnt + NB;                                // [NB] reserved global offset
  std::uint32_t* s_off = s_base + NB;                                // [NB] CTA-local bucket offset
  uint2* s_stage = reinterpret_cast<uint2*>(s_dyn8 + (3 * NB + 1) / 2);  // [kScatterItems]
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t total = p.count[mb];
  const std::uint32_t c0 = blockIdx.x * kScatterItems;
  if (c0 >= total) return;
  const std::uint32_t nloc = min(kScatterItems, total - c0);
  const std::uint32_t* ids = p.ids + mb * p.ids_stride;
  std::uint32_t v[kPer], lr[kPer];
#pragma unroll
  for (std::uint32_t k = 0; k < kPer; ++k) {
    const std::uint32_t i = c0 + threadIdx.x + k * kBktThreads;
    v[k] = i < total ? __ldg(ids + i) : 0xffffffffu;
  }
  for (std::uint32_t b = threadIdx.x; b < NB; b += kBktThreads) s_cnt[b] = 0;
  __syncthreads();
#pragma unroll
  for (std::uint32_t k = 0; k < kPer; ++k)
    if (v[k] != 0xffffffffu) lr[k] = atomicAdd(&s_cnt[v[k] >> p.bb], 1u);
  __syncthreads();
  {
    const std::uint32_t per = (NB + kBktThreads - 1) / kBktThreads;
    const std::uint32_t b0 = min(NB, threadIdx.x * per), b1 = min(NB, b0 + per);
    unsigned long long mine = 0, tot;
    for (std::uint32_t b = b0; b < b1; ++b) mine += s_cnt[b];
    std::uint32_t run = (std::uint32_t)(block_inclusive_scan<kBktThreads>(mine, s_sm, &tot) - mine);
    std::uint32_t* cur = p.cursor + (std::uint64_t)mb * NB;
    for (std::uint32_t b = b0; b < b1; ++b) {
      const std::uint32_t c = s_cnt[b];
      s_off[b] = run;
      run += c;
      if (c) s_base[b] = atomicAdd(cur + b, c);
    }
  }
  __syncthreads();
#pragma unroll
  for (std::uint32_t k = 0; k < kPer; ++k)
    if (v[k] != 0xffffffffu) s_stage[s_off[v[k] >> p.bb] + lr[k]] = make_uint2(v[k], c0 + threadIdx.x + k * kBktThreads);
  __syncthreads();
  uint2* out = p.pairs + mb * p.pair_stride;
  for (std::uint32_t i = threadIdx.x; i < nloc; i += kBktThreads) {
    const uint2 q = s_stage[i];
    const std::uint32_t b = q.x >> p.bb;
    out[s_base[b] + (i - s_off[b])] = q;
  }
}

struct DedupParams {
  BucketParams bp;
  std::uint32_t nmb;
  std::uint32_t* list;  // F_h or all_vertices [M][cap_list]
  std::uint64_t cap_list;
  std::uint32_t* count;  // |F_h| or |all| [M]
  // hop level: dst[mb * dst_stride + tag] = rank (MFG relabel)
  std::uint32_t* dst;
  std::uint64_t dst_stride;
  // every level: base[mb][b] = rank of bucket b's first vertex in the list
  // ([M][NB + 1]); the all level ranges F_1..F_L with the hops' bases
  std::uint32_t* base_out;
  const std::uint32_t* fbase[VK_MAX_HOPS + 1];  // all level: hop h's bases
  std::uint32_t* allidx[VK_MAX_HOPS + 1];
  // next hop's MFG row pointers over the list (HAS_NEXT)
  const std::uint32_t* outdeg;
  std::uint32_t f_next;
  std::uint32_t* indptr_next;  // [M][cap_list + 1]
  std::uint32_t* ecount_next;  // [M]
};

constexpr std::uint32_t kDegStage = 1024;  // capped degrees staged per bucket (else reloaded)
constexpr std::uint32_t kPairRegs = 8;     // pairs per thread kept in registers between passes
constexpr std::uint32_t kMbGroup = 8;      // minibatches interleaved per block group (L2 footprint)

// Shared memory of a dedup CTA: the bucket bitmap (BW words), each word's
// global rank, and (hop levels with a next hop) staged capped degrees.
// Words are padded by one per thread-owned run of wpt words (index
// w + w / wpt), so the owner threads' strided passes are bank-conflict free.
__host__ __device__ constexpr std::size_t dedup_smem(std::uint32_t bb, bool degrees) {
  return (((std::size_t)1 << (bb - 6)) + kBktThreads) * 12 + (degrees ? kDegStage * 4 : 0);
}

// The bucket bitmap and per-word ranks in shared memory (padded layout).
struct SBits {
  unsigned long long* bits;
  std::uint32_t* rank;
  std::uint32_t lw;  // log2(words per thread)
  __device__ __forceinline__ std::uint32_t idx(std::uint32_t w) const { return w + (w >> lw); }
  __device__ __forceinline__ void set(std::uint32_t v) const {
    atomicOr(reinterpret_cast<unsigned*>(bits) + 2 * idx(v >> 6) + ((v >> 5) & 1u), 1u << (v & 31));
  }
  // rank of a present v, once rank[] holds the global rank of every nonzero word
  __device__ __forceinline__ std::uint32_t rank_of(std::uint32_t v) const {
    const std::uint32_t i = idx(v >> 6);
    return rank[i] + (std::uint32_t)__popcll(bits[i] & ((1ull << (v & 63)) - 1ull));
  }
};

// blockIdx -> (minibatch, bucket): groups of kMbGroup minibatches, buckets
// ascending, minibatch fastest inside a group. Blocks are dispatched in
// index order, so every look-back predecessor (same minibatch, lower bucket)
// has a lower index and is already resident or done; a group's random writes
// (MFG dst) stay inside a few minibatches' rows, i.e. inside L2.
__device__ __forceinline__ bool dedup_coords(std::uint32_t nmb, std::uint32_t NB, std::uint32_t& mb,
                                             std::uint32_t& b) {
  // grid (kMbGroup * NB, ceil(nmb / kMbGroup)); the last group may be partial,
  // its surplus blocks exit
  const std::uint32_t g = blockIdx.y;
  const std::uint32_t gsize = min(kMbGroup, nmb - g * kMbGroup);
  if (gsize == kMbGroup) {
    b = blockIdx.x / kMbGroup;
    mb = g * kMbGroup + blockIdx.x % kMbGroup;
  } else {
    b = blockIdx.x / gsize;
    mb = g * kMbGroup + blockIdx.x % gsize;
  }
  return b < NB;
}

struct BitCursor {
  std::uint32_t w0, p0;  // first word of the thread, its padded index
  unsigned m;            // its nonzero words not yet visited (bit k = word w0 + k)
  unsigned long long x;  // remaining bits of the current word
  std::uint32_t w;       // current word
  __device__ __forceinline__ int next8(const unsigned long long* bits, std::uint32_t* vv) {
    int nq = 0;
    while (nq < 8) {
      if (!x) {
        if (!m) break;
        const std::uint32_t k = __ffs((int)m) - 1;
        m &= m - 1;
        w = w0 + k;
        x = bits[p0 + k];
      }
      const int b = __ffsll(x) - 1;
      x &= x - 1;
      vv[nq++] = w * 64 + b;
    }
    return nq;
  }
};

// Zero the padded bitmap; returns the view. wpt = words per thread.
__device__ __forceinline__ SBits sbits_init(unsigned long long* smem, std::uint32_t BW, std::uint32_t wpt) {
  const std::uint32_t BWp = BW + kBktThreads;
  SBits sb{smem, reinterpret_cast<std::uint32_t*>(smem + BWp), (std::uint32_t)(__ffs((int)wpt) - 1)};
  for (std::uint32_t w = threadIdx.x; w < BWp; w += kBktThreads) smem[w] = 0ull;
  return sb;
}

// This thread's wpt consecutive words (<= 32, padded run at p0): distinct
// count and the mask of nonzero words, the only ones later passes visit.
__device__ __forceinline__ unsigned long long count_words(const SBits& sb, std::uint32_t p0, std::uint32_t wpt,
                                                          unsigned& nz) {
  unsigned long long vc = 0;
  nz = 0;
#pragma unroll 1
  for (std::uint32_t k = 0; k < wpt; ++k) {
    const unsigned long long x = sb.bits[p0 + k];
    if (x) {
      nz |= 1u << k;
      vc += __popcll(x);
    }
  }
  return vc;
}

// 4a. hop level: one CTA per (minibatch, bucket) over that bucket's pairs.
template <bool HAS_NEXT>
__global__ void __launch_bounds__(kBktThreads, 4) k_bucket_dedup_hop(DedupParams p) {
  extern __shared__ unsigned long long s_dd[];
  __shared__ unsigned long long s_sm[kBktThreads / 32];
  __shared__ unsigned long long s_excl;
  const BucketParams& bp = p.bp;
  const std::uint32_t NB = bp.NB, BW = 1u << (bp.bb - 6), wpt = BW / kBktThreads;
  std::uint32_t mb, b;
  if (!dedup_coords(p.nmb, NB, mb, b)) return;
  const std::uint32_t* bs = bp.bstart + (std::uint64_t)mb * (NB + 1);
  const std::uint32_t s = bs[b], e = bs[b + 1];
  unsigned long long* status = bp.status + (std::uint64_t)mb * NB;
  const bool last = b + 1 == NB;
  const uint2* pairs = bp.pairs + mb * bp.pair_stride;
  // this thread's pairs, in flight while the bitmap is cleared (kept for the rank pass)
  uint2 pr[kPairRegs];
#pragma unroll
  for (std::uint32_t k = 0; k < kPairRegs; ++k) {
    const std::uint32_t i = s + threadIdx.x + k * kBktThreads;
    pr[k] = i < e ? pairs[i] : make_uint2(0u, 0u);
  }
  const SBits sb = sbits_init(s_dd, BW, wpt);
  std::uint32_t* s_deg = sb.rank + BW + kBktThreads;
  __syncthreads();
  const std::uint32_t vbase = b << bp.bb;
#pragma unroll
  for (std::uint32_t k = 0; k < kPairRegs; ++k)
    if (s + threadIdx.x + k * kBktThreads < e) sb.set(pr[k].x - vbase);
  for (std::uint32_t i = s + threadIdx.x + kPairRegs * kBktThreads; i < e; i += kBktThreads) sb.set(pairs[i].x - vbase);
  __syncthreads();
  const std::uint32_t w0 = threadIdx.x * wpt, p0 = w0 + threadIdx.x;
  unsigned nz;
  const unsigned long long vc = count_words(sb, p0, wpt, nz);
  unsigned long long vtot;
  const std::uint32_t lpos = (std::uint32_t)(block_inclusive_scan<kBktThreads>(vc, s_sm, &vtot) - vc);
  unsigned long long dc = 0, dlex = 0, dtot = 0;
  if (HAS_NEXT) {
    // next hop's row lengths min(f, deg): every degree of the CTA in flight
    // in batches of 8, staged in shared memory by bucket-local position
    BitCursor c{w0, p0, nz, 0ull, 0u};
    std::uint32_t pos = lpos;
    while (true) {
      std::uint32_t vv[8], d[8];
      const int nq = c.next8(sb.bits, vv);
      if (!nq) break;
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = q < nq ? __ldg(p.outdeg + vbase + vv[q]) : 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nq) {
          const std::uint32_t cd = min(p.f_next, d[q]);
          if (pos < kDegStage) s_deg[pos] = cd;
          ++pos;
          dc += cd;
        }
    }
    dlex = block_inclusive_scan<kBktThreads>(dc, s_sm, &dtot) - dc;
  }
  const unsigned long long total = pack_vd(vtot, dtot);
  if (threadIdx.x < 32) {
    const unsigned long long ex = lookback_warp(status, b, total);
    if (threadIdx.x == 0) s_excl = ex;
  }
  __syncthreads();
  const unsigned long long base = s_excl;
  std::uint32_t gv = (std::uint32_t)unpack_v(base) + lpos;
  std::uint32_t gd = (std::uint32_t)(unpack_d(base) + dlex);
  std::uint32_t* list = p.list + mb * p.cap_list;
  std::uint32_t* ipn = HAS_NEXT ? p.indptr_next + mb * (p.cap_list + 1) : nullptr;
  std::uint32_t pos = lpos;
  for (unsigned m = nz; m; m &= m - 1) {  // ranks are only looked up in nonzero words
    const std::uint32_t k = __ffs((int)m) - 1;
    sb.rank[p0 + k] = gv;
    unsigned long long x = sb.bits[p0 + k];
    while (x) {
      const std::uint32_t v = vbase + (w0 + k) * 64 + (__ffsll(x) - 1);
      x &= x - 1;
      list[gv++] = v;
      if (HAS_NEXT) {
        ipn[gv - 1] = gd;
        gd += pos < kDegStage ? s_deg[pos] : min(p.f_next, __ldg(p.outdeg + v));
        ++pos;
      }
    }
  }
  std::uint32_t* bo = p.base_out + (std::uint64_t)mb * (NB + 1);
  if (threadIdx.x == 0) bo[b] = (std::uint32_t)unpack_v(base);
  if (last && threadIdx.x == kBktThreads - 1) {
    const unsigned long long all = base + total;
    const std::uint32_t tv = (std::uint32_t)unpack_v(all), td = (std::uint32_t)unpack_d(all);
    p.count[mb] = tv;
    bo[NB] = tv;
    if (HAS_NEXT) {
      ipn[tv] = td;
      p.ecount_next[mb] = td;
    }
  }
  __syncthreads();
  std::uint32_t* dst = p.dst + mb * p.dst_stride;
#pragma unroll
  for (std::uint32_t k = 0; k < kPairRegs; ++k)
    if (s + threadIdx.x + k * kBktThreads < e) dst[pr[k].y] = sb.rank_of(pr[k].x - vbase);
  for (std::uint32_t i = s + threadIdx.x + kPairRegs * kBktThreads; i < e; i += kBktThreads) {
    const uint2 q = pairs[i];
    dst[q.y] = sb.rank_of(q.x - vbase);
  }
}

// 4b. all level: all_vertices = sorted unique(F_0 u F_1 .. F_L) per bucket.
// F_1..F_L are sorted and their dedups recorded every bucket's index range
// (fbase, same bucket width), so they need no scatter pass and the relabel
// maps are written contiguously; only the batch F_0 (unsorted) goes through
// hist / scan / scatter first.
__global__ void __launch_bounds__(kBktThreads) k_bucket_dedup_all(DedupParams p) {
  extern __shared__ unsigned long long s_dd[];
  __shared__ unsigned long long s_sm[kBktThreads / 32];
  __shared__ unsigned long long s_excl;
  __shared__ std::uint32_t s_lo[VK_MAX_HOPS + 1], s_hi[VK_MAX_HOPS + 1];
  const BucketParams& bp = p.bp;
  const std::uint32_t NB = bp.NB, BW = 1u << (bp.bb - 6), wpt = BW / kBktThreads;
  std::uint32_t mb, b;
  if (!dedup_coords(p.nmb, NB, mb, b)) return;
  const std::uint32_t vbase = b << bp.bb;
  const std::uint32_t vend = (b + 1 == NB) ? 0xffffffffu : vbase + (1u << bp.bb);
  if (threadIdx.x >= 1 && threadIdx.x <= bp.L) {
    const std::uint32_t* fb = p.fbase[threadIdx.x] + (std::uint64_t)mb * (NB + 1);
    s_lo[threadIdx.x] = fb[b];
    s_hi[threadIdx.x] = fb[b + 1];
  }
  // the batch F_0 (unsorted) was bucketed by the hop machinery: pairs
  // {id, index in F_0} of this bucket
  const std::uint32_t* bs = bp.bstart + (std::uint64_t)mb * (NB + 1);
  const std::uint32_t s0 = bs[b], e0 = bs[b + 1];
  const uint2* pairs = bp.pairs + mb * bp.pair_stride;
  const SBits sb = sbits_init(s_dd, BW, wpt);
  __syncthreads();
  // loads issued kBatch at a time ahead of their uses
  constexpr std::uint32_t kBatch = 8;
  auto set_range = [&](const std::uint32_t* F, std::uint32_t lo, std::uint32_t hi, bool filter) {
    for (std::uint32_t i0 = lo + threadIdx.x; i0 < hi; i0 += kBatch * kBktThreads) {
      std::uint32_t v[kBatch];
#pragma unroll
      for (std::uint32_t k = 0; k < kBatch; ++k) {
        const std::uint32_t i = i0 + k * kBktThreads;
        v[k] = i < hi ? __ldg(F + i) : 0xffffffffu;
      }
#pragma unroll
      for (std::uint32_t k = 0; k < kBatch; ++k)
        if (v[k] != 0xffffffffu && (!filter || (v[k] >= vbase && v[k] < vend))) sb.set(v[k] - vbase);
    }
  };
  for (std::uint32_t i = s0 + threadIdx.x; i < e0; i += kBktThreads) sb.set(pairs[i].x - vbase);
  for (std::uint32_t h = 1; h <= bp.L; ++h) set_range(bp.F[h] + mb * bp.capF[h], s_lo[h], s_hi[h], false);
  __syncthreads();
  const std::uint32_t w0 = threadIdx.x * wpt, p0 = w0 + threadIdx.x;
  unsigned nz;
  const unsigned long long vc = count_words(sb, p0, wpt, nz);
  unsigned long long total;
  const std::uint32_t lpos = (std::uint32_t)(block_inclusive_scan<kBktThreads>(vc, s_sm, &total) - vc);
  unsigned long long* status = bp.status + (std::uint64_t)mb * NB;
  const unsigned long long agg = pack_vd(total, 0);
  if (threadIdx.x < 32) {
    const unsigned long long ex = lookback_warp(status, b, agg);
    if (threadIdx.x == 0) s_excl = ex;
  }
  __syncthreads();
  const std::uint32_t base = (std::uint32_t)unpack_v(s_excl);
  std::uint32_t gv = base + lpos;
  std::uint32_t* list = p.list + mb * p.cap_list;
  for (unsigned m = nz; m; m &= m - 1) {
    const std::uint32_t k = __ffs((int)m) - 1;
    sb.rank[p0 + k] = gv;
    unsigned long long x = sb.bits[p0 + k];
    while (x) {
      list[gv++] = vbase + (w0 + k) * 64 + (__ffsll(x) - 1);
      x &= x - 1;
    }
  }
  std::uint32_t* tb = p.base_out + (std::uint64_t)mb * (NB + 1);
  if (threadIdx.x == 0) tb[b] = base;
  if (b + 1 == NB && threadIdx.x == kBktThreads - 1) {
    const std::uint32_t tv = base + (std::uint32_t)total;
    p.count[mb] = tv;
    tb[NB] = tv;
  }
  __syncthreads();
  auto rank_range = [&](const std::uint32_t* F, std::uint32_t* ai, std::uint32_t lo, std::uint32_t hi, bool filter) {
    for (std::uint32_t i0 = lo + threadIdx.x; i0 < hi; i0 += kBatch * kBktThreads) {
      std::uint32_t v[kBatch];
#pragma unroll
      for (std::uint32_t k = 0; k < kBatch; ++k) {
        const std::uint32_t i = i0 + k * kBktThreads;
        v[k] = i < hi ? __ldg(F + i) : 0xffffffffu;
      }
#pragma unroll
      for (std::uint32_t k = 0; k < kBatch; ++k)
        if (v[k] != 0xffffffffu && (!filter || (v[k] >= vbase && v[k] < vend)))
          ai[i0 + k * kBktThreads] = sb.rank_of(v[k] - vbase);
    }
  };
  std::uint32_t* ai0 = p.allidx[0] + mb * bp.capF[0];
  for (std::uint32_t i = s0 + threadIdx.x; i < e0; i += kBktThreads) {
    const uint2 q = pairs[i];
    ai0[q.y] = sb.rank_of(q.x - vbase);
  }
  for (std::uint32_t h = 1; h <= bp.L; ++h)
    rank_range(bp.F[h] + mb * bp.capF[h], p.allidx[h] + mb * bp.capF[h], s_lo[h], s_hi[h], false);
}

// 4c. Small hop levels (at most kSmallLevel drawn ids per minibatch, e.g. C4's
// hop 1 with 15,360): one 1024-thread CTA per minibatch sorts the (id, MFG
// position) pairs (bitonic network over kSmallLevel keys, padded with ~0), so
// no histogram / scatter pass and ~400 near-empty buckets per minibatch become
// one CTA. Thread t holds keys t*16 .. t*16+15 in registers: compare-exchange
// distances below 16 stay in the thread, 16..256 go through warp shuffles,
// and only distances >= 512 (15 of the network's 105 stages) through shared
// memory, laid out [q][t] so every access is conflict-free. Same outputs as
// k_bucket_dedup_hop: sorted distinct F_h, next-hop row pointers, MFG dst,
// and the bucket bases the all level ranges F_h with.
constexpr std::uint32_t kSmallLevel = 16384;
constexpr int kSmallLevelThreads = 1024;

template <bool HAS_NEXT>
__global__ void __launch_bounds__(kSmallLevelThreads) k_small_level(DedupParams p) {
  constexpr std::uint32_t kPer = kSmallLevel / kSmallLevelThreads;  // 16 per thread
  constexpr std::uint32_t T = kSmallLevelThreads;
  extern __shared__ unsigned long long s_key[];  // [kPer][T]: key i = t*kPer + q at q*T + t
  __shared__ unsigned long long s_sm[kSmallLevelThreads / 32];
  const BucketParams& bp = p.bp;
  const std::uint32_t mb = blockIdx.x;
  const std::uint32_t cnt = bp.count[mb];
  const std::uint32_t* ids = bp.ids + mb * bp.ids_stride;
  const std::uint32_t t = threadIdx.x;
  unsigned long long key[kPer];  // id << 32 | position
#pragma unroll
  for (std::uint32_t q = 0; q < kPer; ++q) {
    const std::uint32_t i = t * kPer + q;
    key[q] = i < cnt ? ((unsigned long long)__ldg(ids + i) << 32) | i : ~0ull;
  }
  // element i keeps min(a, partner) iff (i is the lower of the pair) == (its
  // k-block ascends)
  auto cx = [](unsigned long long a, unsigned long long b, bool keep_min) {
    return keep_min ? (a < b ? a : b) : (a < b ? b : a);
  };
  for (std::uint32_t k = 2; k <= kSmallLevel; k <<= 1) {
    std::uint32_t j = k >> 1;
    for (; j >= kPer * 32; j >>= 1) {  // partner in another warp: shared memory
      const std::uint32_t m = j / kPer;
#pragma unroll
      for (std::uint32_t q = 0; q < kPer; ++q) s_key[q * T + t] = key[q];
      __syncthreads();
#pragma unroll
      for (std::uint32_t q = 0; q < kPer; ++q) {
        const std::uint32_t i = t * kPer + q;
        key[q] = cx(key[q], s_key[q * T + (t ^ m)], ((i & j) == 0) == ((i & k) == 0));
      }
      __syncthreads();
    }
    for (; j >= kPer; j >>= 1) {  // partner in another lane of the warp
      const std::uint32_t m = j / kPer;
#pragma unroll
      for (std::uint32_t q = 0; q < kPer; ++q) {
        const std::uint32_t i = t * kPer + q;
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, key[q], m);
        key[q] = cx(key[q], b, ((i & j) == 0) == ((i & k) == 0));
      }
    }
#pragma unroll
    for (std::uint32_t jj = kPer / 2; jj > 0; jj >>= 1) {  // partner in this thread
      if (jj > j) continue;
#pragma unroll
      for (std::uint32_t q = 0; q < kPer; ++q)
        if ((q & jj) == 0) {
          const bool up = ((t * kPer + q) & k) == 0;
          const unsigned long long a = key[q], b = key[q | jj];
          if ((a > b) == up) {
            key[q] = b;
            key[q | jj] = a;
          }
        }
    }
  }
#pragma unroll
  for (std::uint32_t q = 0; q < kPer; ++q) s_key[q * T + t] = key[q];
  __syncthreads();
  auto key_at = [&](std::uint32_t i) { return s_key[(i % kPer) * T + i / kPer]; };
  // ranks: thread t owns sorted positions [t*kPer, (t+1)*kPer)
  const std::uint32_t i0 = threadIdx.x * kPer;
  unsigned long long uc = 0;
#pragma unroll
  for (std::uint32_t q = 0; q < kPer; ++q) {
    const std::uint32_t i = i0 + q;
    if (i < cnt && (i == 0 || (key_at(i) >> 32) != (key_at(i - 1) >> 32))) ++uc;
  }
  unsigned long long utot;
  const std::uint32_t ubase = (std::uint32_t)(block_inclusive_scan<kSmallLevelThreads>(uc, s_sm, &utot) - uc);
  std::uint32_t deg[kPer];
  unsigned long long dc = 0;
  if (HAS_NEXT) {
#pragma unroll
    for (std::uint32_t q = 0; q < kPer; ++q) {
      const std::uint32_t i = i0 + q;
      const bool first = i < cnt && (i == 0 || (key_at(i) >> 32) != (key_at(i - 1) >> 32));
      deg[q] = first ? min(p.f_next, __ldg(p.outdeg + (std::uint32_t)(key_at(i) >> 32))) : 0u;
    }
#pragma unroll
    for (std::uint32_t q = 0; q < kPer; ++q) dc += deg[q];
  }
  unsigned long long dtot = 0;
  const std::uint32_t dbase =
      HAS_NEXT ? (std::uint32_t)(block_inclusive_scan<kSmallLevelThreads>(dc, s_sm, &dtot) - dc) : 0u;
  std::uint32_t* list = p.list + mb * p.cap_list;
  std::uint32_t* ipn = HAS_NEXT ? p.indptr_next + mb * (p.cap_list + 1) : nullptr;
  std::uint32_t* dst = p.dst + mb * p.dst_stride;
  std::uint32_t* bo = p.base_out + (std::uint64_t)mb * (bp.NB + 1);
  // r = distinct ids started so far: a run start takes rank r, a repeat
  // (possibly continuing a run an earlier thread started) rank r - 1
  std::uint32_t r = ubase, d = dbase;
#pragma unroll
  for (std::uint32_t q = 0; q < kPer; ++q) {
    const std::uint32_t i = i0 + q;
    if (i >= cnt) break;
    const std::uint32_t v = (std::uint32_t)(key_at(i) >> 32);
    const bool first = i == 0 || (key_at(i - 1) >> 32) != v;
    if (first) {
      list[r] = v;
      if (HAS_NEXT) {
        ipn[r] = d;
        d += deg[q];
      }
      // bucket bases: buckets (previous id's bucket, this bucket] start here
      const std::uint32_t bcur = v >> bp.bb;
      const std::uint32_t bprev = i == 0 ? 0u : (std::uint32_t)(key_at(i - 1) >> 32 >> bp.bb) + 1u;
      for (std::uint32_t bb_ = (i == 0 ? 0u : bprev); bb_ <= bcur; ++bb_) bo[bb_] = r;
      ++r;
    }
    dst[(std::uint32_t)key_at(i)] = r - 1;
  }
  if (threadIdx.x == kSmallLevelThreads - 1) {
    const std::uint32_t U = (std::uint32_t)utot;
    const std::uint32_t blast = cnt ? (std::uint32_t)(key_at(cnt - 1) >> 32 >> bp.bb) + 1u : 0u;
    for (std::uint32_t bb_ = blast; bb_ <= bp.NB; ++bb_) bo[bb_] = U;
    p.count[mb] = U;
    if (HAS_NEXT) {
      ipn[U] = (std::uint32_t)dtot;
      p.ecount_next[mb] = (std::uint32_t)dtot;
    }
  }
}

}  // namespace
}  // namespace vk
