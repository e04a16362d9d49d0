// VIP analysis on the device: hop-wise vertex-inclusion-probability
// propagation in the log(1-p) domain (replaces vipkit::propagate,
// /root/reference/proj/src/vip.cpp:37-83).
//
// Formulation (verified bitwise-equal on CPU):
//   lm_h[v]  = log1p(-w_h(outdeg v) * p_{h-1}[v])        (one value per sampler;
//              the reference evaluates log1p per edge, vip.cpp:66-70)
//   hop_h[u] = clamp(-expm1( sum_{v in in(u)} lm_h[v] ))  (pull over reverse CSR)
//   total[u] = clamp(-expm1( sum_h log1p(-hop_h[u]) ))    (vip.cpp:76-81; the
//              running sum is carried in hop order so it is bit-identical to
//              the reference given the same hop values)
// Only the summation order of the pull differs from the reference, hence the
// 1e-5 relative tolerance of the north-star (exact for the 0/1 special cases).
//
// Kernel shape: rows are grouped by in-degree class; a class is processed by
// G-lane groups (G = 4 .. 32) or whole CTAs; rows above kSplitDeg are cut into
// edge chunks reduced by separate CTAs and finished in fixed chunk order
// (deterministic). The hoist of the next hop, the running total and the hop
// output are fused into the pull's epilogue, so each hop is one pass over the
// reverse CSR. `C` columns (partitions) are propagated together: one index
// stream serves C probability vectors (the lm gather fetches C contiguous
// doubles).
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "internal.cuh"

namespace vk {
namespace {

constexpr double kFlushBelow = 1e-300;  // vip.cpp:16
std::atomic<int> g_lm_force{0};  // 0 automatic, 32 / 64 forced storage width of the hoisted terms
constexpr int kMaxHops = VK_MAX_HOPS;

// In-degree classes: [0] G=4 deg<=12, [1] G=8 <=48, [2] G=16 <=160,
// [3] G=32 <=1536, [4] CTA <=kSplitDeg, [5] split rows (chunked).
constexpr std::uint64_t kClassMax[5] = {12, 48, 160, 1536, 32768};
constexpr std::uint64_t kSplitDeg = 32768;
constexpr std::uint64_t kChunk = 16384;
constexpr int kCtaThreads = 256;
constexpr std::uint64_t kLmDoubleBudget = 64ull << 20;  // double lm kept while [n][C] fits 64 MB

__device__ __forceinline__ double clamp_prob(double x) {  // vip.cpp:18-21
  if (!(x > kFlushBelow)) return 0.0;
  return x < 1.0 ? x : 1.0;
}

struct HopParams {
  const std::uint64_t* off;   // reverse offsets
  const std::uint32_t* tgt;   // reverse targets
  const std::uint32_t* outdeg;
  const void* lm;             // [n][C] current hop, LM (double, or float for large graphs)
  void* lm_next;              // [n][C] next hop (unused on last hop)
  unsigned* unsafe;           // set when a nonzero w*p underflows the float lm storage
  double* hop_out;            // base for column c: hop_out + c*hop_col_stride + (h-1)*n
  double* total;              // [c*n + u] running log-sum, final total on the last hop
  std::uint64_t n;
  std::uint64_t hop_col_stride;  // L*n (0 if hop_out null)
  std::uint32_t h;               // 1-based hop
  std::uint32_t L;
  double f_next;                 // fanout of hop h+1 (as double)
  int write_hop;
  // active sources of this hop (bit v: some column of lm[v] is nonzero), or
  // null: a sparse hop (hop 1: only the train vertices) skips the random lm
  // gathers of inactive sources -- their terms are exactly zero
  const std::uint32_t* active;
};

template <class LM>
__device__ __forceinline__ void store_lm(const HopParams& p, void* dst, std::uint64_t i, double wp);
__device__ __forceinline__ double log1p_neg_fast(double x);

template <class LM>
__device__ __forceinline__ void store_lm(const HopParams& p, void* dst, std::uint64_t i, double wp) {
  const double x = sizeof(LM) == 4 ? log1p_neg_fast(wp) : log1p(-wp);
  if constexpr (sizeof(LM) == 4) {
    // below FLT_MIN the float copy of log1p(-wp) ~ -wp loses relative accuracy:
    // flag it, and the host reruns the propagation with double storage
    if (wp != 0.0 && wp < 1e-37) atomicOr(p.unsafe, 1u);
  }
  static_cast<LM*>(dst)[i] = (LM)x;
}

// Float-storage mode evaluates the epilogue's transcendentals in float
// (relative error ~1e-7, inside the 1e-5 contract); tiny arguments take the
// first-order form, which is exact to 1e-30 relative and keeps values far
// below FLT_MIN. Double-storage mode (small graphs, the exact reference
// checks) keeps the double functions.
__device__ __forceinline__ double neg_expm1_fast(double s) {  // -expm1(s), s <= 0
  if (s > -1e-30) return -s;
  return -(double)expm1f((float)s);
}
__device__ __forceinline__ double log1p_neg_fast(double x) {  // log1p(-x), 0 <= x <= 1
  if (x < 1e-30) return -x;
  return (double)log1pf(-(float)x);
}

// TransitionModel::weight (vip.hpp:22-26) of sampler u for the next hop.
__device__ __forceinline__ double next_weight(const HopParams& p, std::uint64_t u) {
  const double d = (double)p.outdeg[u];
  return d <= p.f_next ? 1.0 : p.f_next / d;
}

template <int C, class LM>
__device__ __forceinline__ void epilogue(const HopParams& p, std::uint64_t u, int c, double s, double w) {
  constexpr bool kFast = sizeof(LM) == 4;
  const double cur = clamp_prob(kFast ? neg_expm1_fast(s) : -expm1(s));
  if (p.write_hop) p.hop_out[c * p.hop_col_stride + (std::uint64_t)(p.h - 1) * p.n + u] = cur;
  double* acc = p.total + (std::uint64_t)c * p.n + u;
  const double term = kFast ? log1p_neg_fast(cur) : log1p(-cur);
  const double a = p.h == 1 ? term : (*acc + term);
  if (p.h == p.L) {
    *acc = clamp_prob(kFast ? neg_expm1_fast(a) : -expm1(a));
  } else {
    *acc = a;
    const double wp = cur == 0.0 ? 0.0 : w * cur;  // vip.cpp:58-60
    store_lm<LM>(p, p.lm_next, u * C + c, wp);
  }
}

// Accumulator of a pull: float when the lm terms are stored in float. The
// sums are tree-shaped (4-term batches, per-lane batches, log2 lane
// reduction), so the float error stays ~(log2(deg) + batches) x 6e-8 relative.
template <class LM>
using AccT = std::conditional_t<sizeof(LM) == 4, float, double>;

template <int C>
__device__ __forceinline__ void load_lm_f(const void* __restrict__ lmv, std::uint32_t v, float* out) {
  const float* lm = static_cast<const float*>(lmv) + (std::uint64_t)v * C;
  if constexpr (C == 1) {
    out[0] = __ldg(lm);
  } else if constexpr (C == 2) {
    const float2 x = __ldg(reinterpret_cast<const float2*>(lm));
    out[0] = x.x;
    out[1] = x.y;
  } else {
#pragma unroll
    for (int k = 0; k < C / 4; ++k) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(lm) + k);
      out[4 * k] = x.x;
      out[4 * k + 1] = x.y;
      out[4 * k + 2] = x.z;
      out[4 * k + 3] = x.w;
    }
  }
}

template <int C, class LM>
__device__ __forceinline__ void load_lm(const void* __restrict__ lmv, std::uint32_t v, double* out) {
  if constexpr (sizeof(LM) == 4) {
    const float* lm = static_cast<const float*>(lmv) + (std::uint64_t)v * C;
    if constexpr (C == 1) {
      out[0] = __ldg(lm);
    } else if constexpr (C == 2) {
      const float2 x = __ldg(reinterpret_cast<const float2*>(lm));
      out[0] = x.x;
      out[1] = x.y;
    } else {
#pragma unroll
      for (int k = 0; k < C / 4; ++k) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(lm) + k);
        out[4 * k] = x.x;
        out[4 * k + 1] = x.y;
        out[4 * k + 2] = x.z;
        out[4 * k + 3] = x.w;
      }
    }
    return;
  }
  const double* lm = static_cast<const double*>(lmv);
  if constexpr (C == 1) {
    out[0] = __ldg(lm + v);
  } else {
    const double2* q = reinterpret_cast<const double2*>(lm + (std::uint64_t)v * C);
#pragma unroll
    for (int k = 0; k < C / 2; ++k) {
      const double2 x = __ldg(q + k);
      out[2 * k] = x.x;
      out[2 * k + 1] = x.y;
    }
  }
}

// Sum of lm over tgt[a..b) for one lane of a G-lane group (stride G, 4 in
// flight).
template <int C, int G, class LM>
__device__ __forceinline__ void lane_sum(const HopParams& p, std::uint64_t a, std::uint64_t b, int lane,
                                         AccT<LM>* s) {
  // batches of 4 predicated index loads, then 4 independent lm gathers: every
  // batch costs two memory round trips, whatever the row's length
  for (std::uint64_t i = a + lane; i < b; i += 4 * G) {
    std::uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i + k * G < b ? __ldg(p.tgt + i + k * G) : 0u;
    bool on[4];  // in range and active (the activity bitmap is small enough to stay in L2)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      on[k] = i + k * G < b && (!p.active || ((__ldg(p.active + (v[k] >> 5)) >> (v[k] & 31)) & 1u));
    if constexpr (sizeof(LM) == 4) {
      // float storage: the 4 terms of a batch are added in float (error
      // ~2e-7 relative, bounded whatever the degree) and converted once
      float x[4][C];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (on[k]) {
          load_lm_f<C>(p.lm, v[k], x[k]);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) x[k][c] = 0.0f;
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) s[c] += (x[0][c] + x[1][c]) + (x[2][c] + x[3][c]);
    } else {
      double x[4][C];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (on[k]) {
          load_lm<C, LM>(p.lm, v[k], x[k]);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) x[k][c] = 0.0;
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) s[c] += (x[0][c] + x[1][c]) + (x[2][c] + x[3][c]);
    }
  }
}

// G-lane groups, one row per group; warp-uniform outer loop so the shuffle
// reduction always runs with the full warp.
template <int C, int G, class LM>
__global__ void __launch_bounds__(256) k_pull_group(HopParams p, const std::uint32_t* __restrict__ rows,
                                                    std::uint64_t nrows) {
  constexpr int kGroupsPerWarp = 32 / G;
  const int lane = threadIdx.x % G;
  const std::uint64_t warp = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) / 32;
  const std::uint64_t nwarps = ((std::uint64_t)gridDim.x * blockDim.x) / 32;
  const int gw = (threadIdx.x % 32) / G;
  // the next row's id and offsets are fetched while this row is summed
  std::uint64_t r0 = warp * kGroupsPerWarp;
  std::uint32_t u = 0;
  std::uint64_t ra = 0, rb = 0;
  if (r0 + gw < nrows) {
    u = rows[r0 + gw];
    ra = p.off[u];
    rb = p.off[u + 1];
  }
  for (; r0 < nrows; r0 += nwarps * kGroupsPerWarp) {
    const std::uint64_t r = r0 + gw;
    const std::uint64_t rn = r + nwarps * kGroupsPerWarp;
    std::uint32_t un = 0;
    std::uint64_t na = 0, nb = 0;
    if (rn < nrows) {
      un = rows[rn];
      na = p.off[un];
      nb = p.off[un + 1];
    }
    AccT<LM> s[C];
#pragma unroll
    for (int c = 0; c < C; ++c) s[c] = 0;
    if (r < nrows) lane_sum<C, G, LM>(p, ra, rb, lane, s);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < C; ++c) s[c] += __shfl_xor_sync(0xffffffffu, s[c], o, G);
    if (r < nrows) {
      const double w = p.h < p.L ? next_weight(p, u) : 1.0;
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (c % G == lane) epilogue<C, LM>(p, u, c, s[c], w);
    }
    u = un;
    ra = na;
    rb = nb;
  }
}

template <int C, class T>
__device__ __forceinline__ void block_reduce(T* s, T (*sh)[C]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < C; ++c) s[c] += __shfl_xor_sync(0xffffffffu, s[c], o);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < C; ++c) sh[w][c] = s[c];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      T t = 0;
      for (int k = 0; k < kCtaThreads / 32; ++k) t += sh[k][c];
      s[c] = t;
    }
  }
  __syncthreads();
}

// One CTA per row (heavy rows).
template <int C, class LM>
__global__ void __launch_bounds__(kCtaThreads) k_pull_cta(HopParams p, const std::uint32_t* __restrict__ rows,
                                                          std::uint64_t nrows) {
  __shared__ AccT<LM> sh[kCtaThreads / 32][C];
  for (std::uint64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const std::uint32_t u = rows[r];
    AccT<LM> s[C];
#pragma unroll
    for (int c = 0; c < C; ++c) s[c] = 0;
    lane_sum<C, kCtaThreads, LM>(p, p.off[u], p.off[u + 1], threadIdx.x, s);
    block_reduce<C, AccT<LM>>(s, sh);
    if (threadIdx.x == 0) {
      const double w = p.h < p.L ? next_weight(p, u) : 1.0;
#pragma unroll
      for (int c = 0; c < C; ++c) epilogue<C, LM>(p, u, c, s[c], w);
    }
  }
}

// Split rows: chunk j covers [chunk_lo[j], chunk_hi[j]) of one row; partial
// sums are reduced in chunk order by k_split_finish.
template <int C, class LM>
__global__ void __launch_bounds__(kCtaThreads) k_pull_chunk(HopParams p, const std::uint64_t* __restrict__ lo,
                                                            const std::uint64_t* __restrict__ hi,
                                                            std::uint64_t nchunks, double* __restrict__ partial) {
  __shared__ AccT<LM> sh[kCtaThreads / 32][C];
  for (std::uint64_t j = blockIdx.x; j < nchunks; j += gridDim.x) {
    AccT<LM> s[C];
#pragma unroll
    for (int c = 0; c < C; ++c) s[c] = 0;
    lane_sum<C, kCtaThreads, LM>(p, lo[j], hi[j], threadIdx.x, s);
    block_reduce<C, AccT<LM>>(s, sh);
    if (threadIdx.x == 0)
#pragma unroll
      for (int c = 0; c < C; ++c) partial[j * C + c] = (double)s[c];
  }
}

template <int C, class LM>
__global__ void k_split_finish(HopParams p, const std::uint32_t* __restrict__ rows,
                               const std::uint64_t* __restrict__ first_chunk, std::uint64_t nrows,
                               const double* __restrict__ partial) {
  const std::uint64_t r = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (std::uint64_t j = first_chunk[r]; j < first_chunk[r + 1]; ++j) s += partial[j * C + c];
    epilogue<C, LM>(p, rows[r], c, s, p.h < p.L ? next_weight(p, rows[r]) : 1.0);
  }
}

// Hop-1 hoist from p0 (vip.cpp:57-61 with log1p moved here) + p0 range check
// (vip.cpp:41-43).
template <int C, class LM>
__global__ void k_hoist_p0(const double* __restrict__ p0, std::uint64_t n, std::uint64_t col0,
                           const std::uint32_t* __restrict__ outdeg, double f1, HopParams hp,
                           unsigned* __restrict__ bad) {
  for (std::uint64_t v = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (std::uint64_t)gridDim.x * blockDim.x) {
    const double d = (double)outdeg[v];
    const double w = d <= f1 ? 1.0 : f1 / d;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double pv = p0[(col0 + c) * n + v];
      if (!(pv >= 0.0 && pv <= 1.0)) *bad = 1u;
      const double wp = pv == 0.0 ? 0.0 : w * pv;
      store_lm<LM>(hp, hp.lm_next, v * C + c, wp);
    }
  }
}

// Activity bitmap of a hop's hoisted terms: bit v = some column of lm[v] is
// nonzero; counts the active vertices.
template <int C, class LM>
__global__ void k_lm_active(const void* __restrict__ lmv, std::uint64_t n, std::uint32_t* __restrict__ bits,
                            unsigned long long* __restrict__ count) {
  const LM* lm = static_cast<const LM*>(lmv);
  unsigned long long cnt = 0;
  const std::uint64_t words = (n + 31) / 32;
  for (std::uint64_t w = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; w < words;
       w += (std::uint64_t)gridDim.x * blockDim.x) {
    std::uint32_t m = 0;
    for (int b = 0; b < 32; ++b) {
      const std::uint64_t v = w * 32 + b;
      if (v >= n) break;
      bool on = false;
#pragma unroll
      for (int c = 0; c < C; ++c) on |= lm[v * C + c] != (LM)0;
      m |= (std::uint32_t)on << b;
    }
    bits[w] = m;
    cnt += __popc(m);
  }
  cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(count, cnt);
}

unsigned grid_cap(int device, std::uint64_t work, unsigned block) {
  const std::uint64_t g = (work + block - 1) / block;
  const std::uint64_t cap = (std::uint64_t)sm_count(device) * (2048 / block) * 4;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <int C, class LM>
void run_columns(vk_graph_s& g, const std::uint32_t* fan, std::uint32_t L, const double* p0_dev,
                 std::uint64_t col0, double* hop_dev, double* total_dev, cudaStream_t st, DevBuf& lm_a,
                 DevBuf& lm_b, DevBuf& partial, const DevBuf& bad) {
  const std::uint64_t n = g.n;
  void* lm = lm_a.p;
  void* lmn = lm_b.p;
  unsigned* unsafe = bad.as<unsigned>() + 1;
  {
    HopParams hp{};
    hp.lm_next = lm;
    hp.unsafe = unsafe;
    k_hoist_p0<C, LM><<<grid_cap(g.device, n, 256), 256, 0, st>>>(p0_dev, n, col0, g.out_deg.as<std::uint32_t>(),
                                                                   (double)fan[0], hp, bad.as<unsigned>());
  }
  count_launch();
  VK_LAUNCH_CHECK();
  const auto& so = g.sched_offsets;  // [6 classes + split-rows meta]
  const std::uint32_t* rows = g.sched_rows.as<std::uint32_t>();
  // source activity: while a hop's active sources are a minority (hop 1 =
  // the partitions' train vertices), its pull skips the inactive ones' lm
  // gathers; once a hop is mostly active the check stops (activity only
  // spreads hop by hop)
  const std::uint64_t words = (n + 31) / 32;
  if (g.vip_active.bytes < words * 4 + 16) g.vip_active.alloc(words * 4 + 16);
  std::uint32_t* act = g.vip_active.as<std::uint32_t>();
  unsigned long long* act_cnt = reinterpret_cast<unsigned long long*>(act + ((words + 1) & ~1ull));
  bool track = true;
  auto activity = [&](const void* lmh) -> const std::uint32_t* {
    if (!track) return nullptr;
    VK_CUDA(cudaMemsetAsync(act_cnt, 0, 8, st));
    k_lm_active<C, LM><<<grid_cap(g.device, words, 256), 256, 0, st>>>(lmh, n, act, act_cnt);
    count_launch();
    VK_LAUNCH_CHECK();
    unsigned long long c = 0;
    VK_CUDA(cudaMemcpyAsync(&c, act_cnt, 8, cudaMemcpyDeviceToHost, st));
    VK_CUDA(cudaStreamSynchronize(st));
    track = c * 2 < n;
    return track ? act : nullptr;
  };
  for (std::uint32_t h = 1; h <= L; ++h) {
    HopParams p;
    p.active = activity(lm);
    p.off = g.rev_off;
    p.tgt = g.rev_tgt;
    p.outdeg = g.out_deg.as<std::uint32_t>();
    p.lm = lm;
    p.lm_next = lmn;
    p.unsafe = unsafe;
    p.hop_out = hop_dev ? hop_dev + col0 * (std::uint64_t)L * n : nullptr;
    p.total = total_dev + col0 * n;
    p.n = n;
    p.hop_col_stride = (std::uint64_t)L * n;
    p.h = h;
    p.L = L;
    p.f_next = h < L ? (double)fan[h] : 1.0;
    p.write_hop = hop_dev != nullptr;
    auto cls = [&](int c) { return std::pair<const std::uint32_t*, std::uint64_t>(rows + so[c], so[c + 1] - so[c]); };
    {
      auto [r, k] = cls(0);
      if (k) k_pull_group<C, 4, LM><<<grid_cap(g.device, k * 4, 256), 256, 0, st>>>(p, r, k), count_launch();
    }
    {
      auto [r, k] = cls(1);
      if (k) k_pull_group<C, 8, LM><<<grid_cap(g.device, k * 8, 256), 256, 0, st>>>(p, r, k), count_launch();
    }
    {
      auto [r, k] = cls(2);
      if (k) k_pull_group<C, 16, LM><<<grid_cap(g.device, k * 16, 256), 256, 0, st>>>(p, r, k), count_launch();
    }
    {
      auto [r, k] = cls(3);
      if (k) k_pull_group<C, 32, LM><<<grid_cap(g.device, k * 32, 256), 256, 0, st>>>(p, r, k), count_launch();
    }
    {
      auto [r, k] = cls(4);
      if (k) {
        const unsigned grid = (unsigned)std::min<std::uint64_t>(k, (std::uint64_t)sm_count(g.device) * 8);
        k_pull_cta<C, LM><<<grid, kCtaThreads, 0, st>>>(p, r, k);
        count_launch();
      }
    }
    {
      auto [r, k] = cls(5);
      if (k) {
        const std::uint64_t nch = so[8];
        const std::uint64_t* meta = reinterpret_cast<const std::uint64_t*>(rows + so[7]);
        // meta layout: lo[nch], hi[nch], first_chunk[k+1]
        const unsigned grid = (unsigned)std::min<std::uint64_t>(nch, (std::uint64_t)sm_count(g.device) * 8);
        k_pull_chunk<C, LM><<<grid, kCtaThreads, 0, st>>>(p, meta, meta + nch, nch, partial.as<double>());
        k_split_finish<C, LM><<<ceil_div(k, 128), 128, 0, st>>>(p, r, meta + 2 * nch, k, partial.as<double>());
        count_launch(2);
      }
    }
    VK_LAUNCH_CHECK();
    std::swap(lm, lmn);
  }
}

}  // namespace

// Build the in-degree class schedule once per graph (host-side bucketing of
// the reverse offsets; one-time cost like the reference's CSR rebuild).
void build_vip_schedule(vk_graph_s& g) {
  if (g.sched_ready) return;
  const std::uint64_t n = g.n;
  std::vector<std::uint64_t> off(n + 1);
  VK_CUDA(cudaMemcpy(off.data(), g.rev_off, (n + 1) * 8, cudaMemcpyDeviceToHost));
  std::vector<std::uint64_t> cnt(6, 0);
  std::vector<std::uint8_t> cls(n);
  std::uint64_t nchunks = 0;
  for (std::uint64_t u = 0; u < n; ++u) {
    const std::uint64_t d = off[u + 1] - off[u];
    int c = 5;
    for (int k = 0; k < 5; ++k)
      if (d <= kClassMax[k]) {
        c = k;
        break;
      }
    cls[u] = (std::uint8_t)c;
    cnt[c]++;
    if (c == 5) nchunks += (d + kChunk - 1) / kChunk;
  }
  // rows (u32) for classes 0..5, then an 8-byte aligned meta block for the
  // split rows: lo[nchunks], hi[nchunks], first_chunk[nsplit+1] (u64).
  std::vector<std::uint64_t> so(9, 0);
  for (int c = 0; c < 6; ++c) so[c + 1] = so[c] + cnt[c];
  std::uint64_t meta_start = (so[6] + 1) & ~1ull;  // u64 alignment in u32 units
  const std::uint64_t nsplit = cnt[5];
  const std::uint64_t meta_words = 2 * nchunks + nsplit + 1;
  std::vector<std::uint32_t> host(meta_start + 2 * meta_words, 0);
  std::vector<std::uint64_t> pos(so.begin(), so.begin() + 6);
  std::vector<std::uint64_t> lo, hi, first{0};
  for (std::uint64_t u = 0; u < n; ++u) {
    host[pos[cls[u]]++] = (std::uint32_t)u;
    if (cls[u] == 5) {
      for (std::uint64_t a = off[u]; a < off[u + 1]; a += kChunk) {
        lo.push_back(a);
        hi.push_back(std::min(off[u + 1], a + kChunk));
      }
      first.push_back(lo.size());
    }
  }
  std::uint64_t* meta = reinterpret_cast<std::uint64_t*>(host.data() + meta_start);
  for (std::uint64_t j = 0; j < nchunks; ++j) {
    meta[j] = lo[j];
    meta[nchunks + j] = hi[j];
  }
  for (std::uint64_t r = 0; r <= nsplit; ++r) meta[2 * nchunks + r] = first[r];
  g.sched_rows.alloc(host.size() * 4);
  VK_CUDA(cudaMemcpy(g.sched_rows.p, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
  so[7] = meta_start;
  so[8] = nchunks;
  g.sched_offsets = so;
  g.sched_ready = true;
}

}  // namespace vk

using namespace vk;

namespace {

void validate_fanouts(const std::uint32_t* fanouts, std::uint32_t L) {
  // FanoutSpec::validate (sampling.cpp:11-15)
  if (L == 0) raise(VK_ERR_PARAMETER, "fanout list must have at least one hop");
  if (L > VK_MAX_HOPS) raise(VK_ERR_UNSUPPORTED, "at most 8 hops are supported");
  if (!fanouts) raise(VK_ERR_PARAMETER, "null fanouts");
  for (std::uint32_t h = 0; h < L; ++h)
    if (fanouts[h] < 1) raise(VK_ERR_PARAMETER, "each fanout must be >= 1");
}

void propagate_device(vk_graph_s& g, const std::uint32_t* fanouts, std::uint32_t L, std::uint32_t ncols,
                      const double* p0, double* hop, double* total, cudaStream_t st) {
  validate_fanouts(fanouts, L);
  if (ncols == 0) return;
  build_vip_schedule(g);
  const std::uint64_t n = g.n;
  const std::uint32_t cmax = ncols >= 8 ? 8 : (ncols >= 4 ? 4 : (ncols >= 2 ? 2 : 1));
  auto ensure = [](DevBuf& b, std::size_t bytes) {
    if (b.bytes < bytes) b.alloc(bytes);
  };
  const std::uint64_t nch = g.sched_offsets[8];
  ensure(g.vip_lm_a, n * 8 * cmax);
  ensure(g.vip_lm_b, n * 8 * cmax);
  ensure(g.vip_partial, std::max<std::uint64_t>(1, nch) * 8 * cmax);
  ensure(g.vip_flag, 2 * sizeof(unsigned));  // [0] p0 out of range, [1] float storage unsafe
  DevBuf& lm_a = g.vip_lm_a;
  DevBuf& lm_b = g.vip_lm_b;
  DevBuf& partial = g.vip_partial;
  DevBuf& bad = g.vip_flag;
  // The hoisted log(1-w*p) terms are stored in float once the double copy
  // would not fit the L2 working-set budget: every random gather then moves
  // half the bytes (and the C=8 row is one 32-byte sector). Accumulation and
  // every output stay double; the float relative error (6e-8 per term, all
  // terms one sign) is far inside the 1e-5 contract. A nonzero term below
  // FLT_MIN sets a flag and the propagation is redone with double storage.
  const int force = g_lm_force.load(std::memory_order_relaxed);  // vk_vip_force_storage
  const bool use_f32 = force == 32 || (force != 64 && n * 8ull * cmax > kLmDoubleBudget);
  auto pass = [&](bool f32) {
    VK_CUDA(cudaMemsetAsync(bad.p, 0, 2 * sizeof(unsigned), st));
    std::uint32_t c0 = 0;
    while (c0 < ncols) {
      const std::uint32_t rem = ncols - c0;
      const std::uint32_t c = rem >= 8 ? 8 : (rem >= 4 ? 4 : (rem >= 2 ? 2 : 1));
      if (f32) {
        if (c == 8) run_columns<8, float>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
        else if (c == 4) run_columns<4, float>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
        else if (c == 2) run_columns<2, float>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
        else run_columns<1, float>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
      } else {
        if (c == 8) run_columns<8, double>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
        else if (c == 4) run_columns<4, double>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
        else if (c == 2) run_columns<2, double>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
        else run_columns<1, double>(g, fanouts, L, p0, c0, hop, total, st, lm_a, lm_b, partial, bad);
      }
      c0 += c;
    }
    unsigned h[2] = {0, 0};
    VK_CUDA(cudaMemcpyAsync(h, bad.p, sizeof h, cudaMemcpyDeviceToHost, st));
    VK_CUDA(cudaStreamSynchronize(st));  // surfaces the p0 range error synchronously
    if (h[0]) raise(VK_ERR_PARAMETER, "p0 entries must lie in [0,1]");
    return h[1] == 0;
  };
  if (!pass(use_f32)) pass(false);
  g.vip_last_f32 = use_f32;
}

}  // namespace

extern "C" {

int vk_initial_probs(uint64_t n, const uint8_t* roles, const uint32_t* part_of, uint32_t k,
                     uint64_t batch_size, double* p0_out) {
  return guard([&] {
    // vip.cpp:25-35
    if (batch_size == 0) raise(VK_ERR_PARAMETER, "batch size must be >= 1");
    if (!roles || !part_of || !p0_out) raise(VK_ERR_PARAMETER, "null argument");
    std::uint64_t T = 0;
    for (std::uint64_t v = 0; v < n; ++v) T += (part_of[v] == k && roles[v] == 0);
    if (T == 0) raise(VK_ERR_SAMPLING, "partition " + std::to_string(k) + " has no train vertices");
    const double p = std::min(1.0, (double)batch_size / (double)T);
    for (std::uint64_t v = 0; v < n; ++v) p0_out[v] = (part_of[v] == k && roles[v] == 0) ? p : 0.0;
  });
}

int vk_vip_force_storage(int bits) {
  return guard([&] {
    if (bits != 0 && bits != 32 && bits != 64) raise(VK_ERR_PARAMETER, "storage width must be 0, 32 or 64");
    g_lm_force.store(bits, std::memory_order_relaxed);
  });
}

int vk_vip_propagate(vk_graph g, const uint32_t* fanouts, uint32_t num_hops, uint32_t ncols,
                     const double* p0, double* hop_out, double* total_out) {
  return guard([&] {
    if (!g || !p0 || !total_out) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(g->device);
    validate_fanouts(fanouts, num_hops);
    const std::uint64_t n = g->n;
    // vip.cpp:41-43 (host-side check keeps the error synchronous and exact)
    for (std::uint64_t i = 0; i < n * (std::uint64_t)ncols; ++i)
      if (!(p0[i] >= 0.0 && p0[i] <= 1.0)) raise(VK_ERR_PARAMETER, "p0 entries must lie in [0,1]");
    DevBuf dp0(n * 8 * ncols), dtot(n * 8 * ncols);
    DevBuf dhop(hop_out ? n * 8 * ncols * num_hops : 0);
    VK_CUDA(cudaMemcpyAsync(dp0.p, p0, n * 8 * ncols, cudaMemcpyHostToDevice, g->stream));
    propagate_device(*g, fanouts, num_hops, ncols, dp0.as<double>(), hop_out ? dhop.as<double>() : nullptr,
                     dtot.as<double>(), g->stream);
    VK_CUDA(cudaMemcpyAsync(total_out, dtot.p, n * 8 * ncols, cudaMemcpyDeviceToHost, g->stream));
    if (hop_out)
      VK_CUDA(cudaMemcpyAsync(hop_out, dhop.p, n * 8 * ncols * num_hops, cudaMemcpyDeviceToHost, g->stream));
    VK_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int vk_vip_propagate_device(vk_graph g, const uint32_t* fanouts, uint32_t num_hops, uint32_t ncols,
                            const double* p0_dev, double* hop_dev, double* total_dev, vk_stream_t stream) {
  return guard([&] {
    if (!g || !p0_dev || !total_dev) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(g->device);
    propagate_device(*g, fanouts, num_hops, ncols, p0_dev, hop_dev, total_dev,
                     stream ? static_cast<cudaStream_t>(stream) : g->stream);
  });
}

}  // extern "C"
