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

// Thread 0 only: publish this tile's aggregate, walk predecessors, publish
// the inclusive prefix, return the exclusive prefix (packed v|d).
__device__ __forceinline__ unsigned long long lookback(unsigned long long* status, unsigned tile,
                                                       unsigned long long aggregate) {
  if (tile == 0) {
    publish(status, kFlagInc | aggregate);
    return 0ull;
  }
  publish(status + tile, kFlagAgg | aggregate);
  unsigned long long ex = 0;
  int t = (int)tile - 1;
  while (true) {
    unsigned long long s;
    do {
      s = peek(status + t);
    } while ((s >> 62) == 0);
    ex += s & kValueMask;
    if ((s >> 62) == 2) break;
    --t;
  }
  publish(status + tile, kFlagInc | (ex + aggregate));
  return ex;
}

}  // namespace vk
