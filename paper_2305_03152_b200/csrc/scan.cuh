// Block-wide scans and the single-pass decoupled look-back used by the
// bitmap compaction (one scan chain per minibatch).
#pragma once
#include <cstdint>

namespace vk {

// Inclusive scan of a u64 across a CTA of NT threads; returns the inclusive
// value and writes the block total to *total. `smem` holds NT/32 u64.
template <int NT>
__device__ __forceinline__ unsigned long long block_inclusive_scan(unsigned long long x,
                                                                   unsigned long long* smem,
                                                                   unsigned long long* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long s = lane < NT / 32 ? smem[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < NT / 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) smem[lane] = s;
  }
  __syncthreads();
  if (w > 0) x += smem[w - 1];
  *total = smem[NT / 32 - 1];
  __syncthreads();
  return x;
}

// Decoupled look-back status word: [63:62] flag (0 empty, 1 aggregate,
// 2 inclusive prefix), [61:31] vertex count (31 bits), [30:0] edge count
// (31 bits). A single 64-bit word, so publication is one store.
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long pack_vd(unsigned long long v, unsigned long long d) {
  return (v << 31) | d;
}
__device__ __forceinline__ unsigned long long unpack_v(unsigned long long x) { return (x >> 31) & 0x7fffffffull; }
__device__ __forceinline__ unsigned long long unpack_d(unsigned long long x) { return x & 0x7fffffffull; }

__device__ __forceinline__ void publish(unsigned long long* st, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(st), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long peek(const unsigned long long* st) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(st) : "memory");
  return v;
}

// Publish this tile's aggregate (tile 0: its inclusive prefix) so that
// successors can look past it; one thread.
__device__ __forceinline__ void publish_aggregate(unsigned long long* status, unsigned tile,
                                                  unsigned long long aggregate) {
  publish(status + tile, (tile == 0 ? kFlagInc : kFlagAgg) | aggregate);
}

// Warp 0 only (all 32 lanes), after publish_aggregate: look back over a
// window of 32 predecessors at a time: the nearest inclusive prefix in the
// window ends the walk, the aggregates after it are summed; lanes whose
// predecessor has not published yet make the warp re-poll. Publishes the
// inclusive prefix and returns the exclusive prefix (packed v|d) to all lanes.
__device__ __forceinline__ unsigned long long lookback_resolve(unsigned long long* status, unsigned tile,
                                                               unsigned long long aggregate) {
  const unsigned lane = threadIdx.x & 31;
  if (tile == 0) return 0ull;
  unsigned long long ex = 0;
  int top = (int)tile - 1;  // highest predecessor not yet accounted for
  while (true) {
    const int t = top - (int)lane;
    unsigned long long s = t >= 0 ? peek(status + t) : (kFlagInc);  // t < 0: virtual zero prefix
    unsigned flag = (unsigned)(s >> 62);
    // wait until every lane's predecessor has published something, backing
    // off between polls: hundreds of spinning warps otherwise hammer the few
    // L2 slices that hold a chain's status words and slow every CTA down
    unsigned ns = 32;
    while (__any_sync(0xffffffffu, flag == 0)) {
      __nanosleep(ns);
      ns = min(ns * 2, 1024u);
      if (flag == 0) {
        s = peek(status + t);
        flag = (unsigned)(s >> 62);
      }
    }
    const unsigned inc_mask = __ballot_sync(0xffffffffu, flag == 2);
    if (inc_mask) {
      const unsigned first = __ffs(inc_mask) - 1;  // nearest inclusive predecessor
      unsigned long long v = lane <= first ? (s & kValueMask) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      ex += v;
      break;
    }
    unsigned long long v = s & kValueMask;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    ex += v;
    top -= 32;
  }
  if (lane == 0) publish(status + tile, kFlagInc | (ex + aggregate));
  return ex;
}

// Warp 0 only: publish the aggregate, then resolve the look-back.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* status, unsigned tile,
                                                            unsigned long long aggregate) {
  if ((threadIdx.x & 31) == 0) publish_aggregate(status, tile, aggregate);
  return lookback_resolve(status, tile, aggregate);
}

// In-place exclusive scan of n u32 values (the last output is the total of
// all earlier inputs): one pass, 2048 values per CTA, decoupled look-back
// across CTAs in blockIdx order. Totals must stay below 2^31.
constexpr int kScanU32Threads = 256, kScanU32Items = 8;
static __global__ void __launch_bounds__(kScanU32Threads) k_scan_u32(std::uint32_t* __restrict__ a, std::uint64_t n,
                                                            unsigned long long* __restrict__ status) {
  __shared__ unsigned long long s_sm[kScanU32Threads / 32];
  __shared__ unsigned long long s_excl;
  const std::uint64_t base = ((std::uint64_t)blockIdx.x * kScanU32Threads + threadIdx.x) * kScanU32Items;
  std::uint32_t x[kScanU32Items];
  unsigned long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanU32Items; ++k) {
    x[k] = base + k < n ? a[base + k] : 0u;
    sum += x[k];
  }
  unsigned long long total;
  const unsigned long long lex = block_inclusive_scan<kScanU32Threads>(sum, s_sm, &total) - sum;
  if (threadIdx.x < 32) {
    const unsigned long long ex = lookback_warp(status, blockIdx.x, pack_vd(total, 0));
    if (threadIdx.x == 0) s_excl = ex;
  }
  __syncthreads();
  unsigned long long run = unpack_v(s_excl) + lex;
#pragma unroll
  for (int k = 0; k < kScanU32Items; ++k)
    if (base + k < n) {
      a[base + k] = (std::uint32_t)run;
      run += x[k];
    }
}

}  // namespace vk
