// NVLink row-exchange microbenchmark (one process, two GPUs, peer access):
// is the miss exchange bound by the link, by read latency, or by contention
// with the HBM-bound gather it overlaps? Rows of 256 B, a sorted random
// subset (the exchange's distinct request list shape) of a 14 GB store.
//   pull   : GPU0 kernel reads GPU1's rows, writes local staging
//   push   : GPU1 kernel reads its rows, writes GPU0's staging
//   memcpy : cudaMemcpyPeerAsync of the same byte count (contiguous)
//   tma    : the pull issued through the TMA engine (cp.async.bulk rows into
//            a shared-memory ring, bulk stores out), 64 threads per SM
//   *2     : both directions at once (each GPU serves the other)
//   +copy  : the same with an HBM copy kernel (the gather's stand-in) running
//            on both GPUs meanwhile; exchange kernels on a high-priority stream
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o nvlink_rows_bench nvlink_rows_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1); } } while (0)

// 16 lanes per 256 B row, U rows per half-warp in flight
template <int U>
__global__ void __launch_bounds__(256) k_rows(const uint4* __restrict__ src, const uint32_t* __restrict__ list,
                                              uint32_t cnt, uint4* __restrict__ dst) {
  const uint32_t hw = (blockIdx.x * blockDim.x + threadIdx.x) >> 4, c = threadIdx.x & 15;
  const uint32_t nhw = (gridDim.x * blockDim.x) >> 4;
  for (uint32_t r0 = hw * U; r0 < cnt; r0 += nhw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < cnt) v[u] = src[(uint64_t)list[r0 + u] * 16 + c];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < cnt) dst[(uint64_t)(r0 + u) * 16 + c] = v[u];
  }
}


// The pull through the TMA engine: per warp a ring of K stages of 32 rows
// (8 KB); each lane issues one 256 B cp.async.bulk load (peer -> shared),
// lane 0 one 8 KB bulk store (shared -> staging) D iterations later. Two
// warps per SM hold ~9.5 MB in flight GPU-wide with 64 threads per SM.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int K, int D, int NW>
__global__ void __launch_bounds__(32 * NW) k_rows_tma(const uint4* __restrict__ src, const uint32_t* __restrict__ list,
                                                     uint32_t cnt, uint4* __restrict__ dst) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* ring = smem + (size_t)w * K * 8192;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + (size_t)NW * K * 8192) + w * K;
  if (lane == 0) {
    for (int s = 0; s < K; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const uint32_t gw = blockIdx.x * NW + w, nw = gridDim.x * NW;
  const uint32_t nch = (cnt + 31) / 32;
  const uint32_t niter = gw < nch ? (nch - gw + nw - 1) / nw : 0;
  for (uint32_t it = 0; it < niter + D; ++it) {
    if (it < niter) {
      const uint32_t c = gw + it * nw, s = it % K, rows = min(32u, cnt - c * 32);
      const uint32_t idx = lane < (int)rows ? list[c * 32 + lane] : 0u;
      const unsigned bar = smem_u32(bars + s);
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K - D - 1) : "memory");  // stage s's old store read
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rows * 256) : "memory");
      }
      __syncwarp();
      if (lane < (int)rows)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(smem_u32(ring + s * 8192 + lane * 256)), "l"(src + (uint64_t)idx * 16), "r"(bar)
                     : "memory");
    }
    if (it >= D && lane == 0) {
      const uint32_t j = it - D, c = gw + j * nw, s = j % K, rows = min(32u, cnt - c * 32);
      const unsigned bar = smem_u32(bars + s), par = (j / K) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(done) : "r"(bar), "r"(par) : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(dst + (uint64_t)c * 32 * 16), "r"(smem_u32(ring + s * 8192)), "r"(rows * 256) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
constexpr int kTK = 8, kTD = 4, kTNW = 2;
constexpr size_t kTmaSmem = (size_t)kTNW * kTK * 8192 + kTNW * kTK * 8;

__global__ void k_fill(uint4* a, uint64_t rows, uint32_t d) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows * 16; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_uint4((uint32_t)(i >> 4), (uint32_t)(i & 15), d, 0xabcdu);
}
// non-persistent, like the gather: 4 vectors per thread, one launch per pass
__global__ void k_copy1(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
  const uint64_t i0 = blockIdx.x * 1024ull + threadIdx.x;
  uint4 v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (i0 + u * 256 < n) v[u] = a[i0 + u * 256];
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (i0 + u * 256 < n) b[i0 + u * 256] = v[u];
}
static void k_copy_launch(const uint4* a, uint4* b, uint64_t n, int reps, cudaStream_t st) {
  for (int r = 0; r < reps; ++r) k_copy1<<<(unsigned)((n + 1023) / 1024), 256, 0, st>>>(a, b, n);
}

int main(int argc, char** argv) {
  const uint64_t store_rows = 55ull << 20, req = argc > 1 ? std::strtoull(argv[1], 0, 10) : 10000000ull;
  const int ctas_per_sm = argc > 2 ? std::atoi(argv[2]) : 2;
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { std::printf("need 2 GPUs\n"); return 1; }
  for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceEnablePeerAccess(1 - d, 0)); }
  std::mt19937_64 g(7);
  std::vector<uint32_t> h(req);
  for (auto& x : h) x = (uint32_t)(g() % store_rows);
  std::sort(h.begin(), h.end());
  uint4 *store[2], *stage[2], *ca[2], *cb[2];
  uint32_t* list[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&store[d], store_rows * 256));
    k_fill<<<148 * 16, 256>>>(store[d], store_rows, d);
    CK(cudaMalloc(&stage[d], req * 256));
    CK(cudaMalloc(&list[d], req * 4));
    CK(cudaMemcpy(list[d], h.data(), req * 4, cudaMemcpyHostToDevice));
  }
  const uint64_t copy_bytes = 4ull << 30;
  cudaStream_t s[2], sc[2];
  cudaEvent_t e0[2], e1[2], cev0[2], cev1[2];
  int plo, phi;
  CK(cudaDeviceGetStreamPriorityRange(&plo, &phi));
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&ca[d], copy_bytes));
    CK(cudaMalloc(&cb[d], copy_bytes));
    CK(cudaStreamCreateWithPriority(&s[d], cudaStreamNonBlocking, phi));
    CK(cudaStreamCreateWithFlags(&sc[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&cev0[d]));
    CK(cudaEventCreate(&cev1[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  CK(cudaSetDevice(0));
  cudaEvent_t c0, c1;
  CK(cudaEventCreate(&c0));
  CK(cudaEventCreate(&c1));
  const double gb = req * 256.0 / 1e9;
  const unsigned grid = 148 * ctas_per_sm;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFuncSetAttribute(k_rows_tma<kTK, kTD, kTNW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  }
  // mode: 0 pull, 1 push, 2 memcpy, 3 pull through TMA; dirs: 1 or 2; with_copy
  auto run = [&](int mode, int dirs, bool with_copy, const char* name) {
    float best[2] = {1e9f, 1e9f}, copy_ms = 0;
    for (int it = 0; it < 4; ++it) {
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      if (with_copy)  // both GPUs run a gather-sized HBM copy (4 x 8 GB r+w) meanwhile
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(cev0[d], sc[d]));
          k_copy_launch(ca[d], cb[d], copy_bytes / 16, 4, sc[d]);
          CK(cudaEventRecord(cev1[d], sc[d]));
        }
      for (int t = 0; t < dirs; ++t) {  // t: requester
        const int req_dev = t, own = 1 - t;
        const int launch_dev = mode == 1 ? own : req_dev;
        CK(cudaSetDevice(launch_dev));
        CK(cudaEventRecord(e0[launch_dev], s[launch_dev]));
        if (mode == 2)
          CK(cudaMemcpyPeerAsync(stage[req_dev], req_dev, store[own], own, req * 256, s[launch_dev]));
        else if (mode == 3)
          k_rows_tma<kTK, kTD, kTNW><<<148, 32 * kTNW, kTmaSmem, s[launch_dev]>>>(store[own], list[launch_dev],
                                                                               (uint32_t)req, stage[req_dev]);
        else
          k_rows<4><<<grid, 256, 0, s[launch_dev]>>>(store[own], list[launch_dev], (uint32_t)req, stage[req_dev]);
        CK(cudaEventRecord(e1[launch_dev], s[launch_dev]));
      }
      for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      CK(cudaGetLastError());
      for (int t = 0; t < dirs; ++t) {
        const int ld = mode == 1 ? 1 - t : t;
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[ld], e1[ld]));
        best[t] = std::min(best[t], ms);
      }
      if (with_copy) {
        float a, b;
        CK(cudaEventElapsedTime(&a, cev0[0], cev1[0]));
        CK(cudaEventElapsedTime(&b, cev0[1], cev1[1]));
        copy_ms = std::max(a, b);
      }
    }
    std::printf("%-22s dir0 %7.3f ms (%6.1f GB/s)", name, best[0], gb / best[0] * 1e3);
    if (dirs == 2) std::printf("  dir1 %7.3f ms (%6.1f GB/s)", best[1], gb / best[1] * 1e3);
    if (with_copy) std::printf("  copies (32 GB r+w each) %7.3f ms (%6.1f GB/s)", copy_ms, 8.0 * copy_bytes / 1e9 / copy_ms * 1e3);
    std::printf("\n");
  };
  std::printf("rows %llu (%.2f GB), grid %u\n", (unsigned long long)req, gb, grid);
  {  // copy alone
    float ms = 0;
    CK(cudaSetDevice(0));
    for (int it = 0; it < 3; ++it) {
      CK(cudaEventRecord(c0, sc[0]));
      k_copy_launch(ca[0], cb[0], copy_bytes / 16, 4, sc[0]);
      CK(cudaEventRecord(c1, sc[0]));
      CK(cudaStreamSynchronize(sc[0]));
      CK(cudaEventElapsedTime(&ms, c0, c1));
    }
    std::printf("%-22s %7.3f ms (%6.1f GB/s)\n", "local copy alone", ms, 8.0 * copy_bytes / 1e9 / ms * 1e3);
  }
  run(2, 1, false, "memcpy peer 1 dir");
  run(2, 2, false, "memcpy peer 2 dir");
  run(0, 1, false, "pull 1 dir");
  run(0, 2, false, "pull 2 dir");
  run(1, 1, false, "push 1 dir");
  run(1, 2, false, "push 2 dir");
  run(3, 1, false, "tma pull 1 dir");
  {  // the TMA pull's staging holds the requested rows
    std::vector<uint4> got(req * 16);
    CK(cudaSetDevice(0));
    CK(cudaMemcpy(got.data(), stage[0], req * 256, cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (uint64_t r = 0; r < req; ++r)
      for (int c = 0; c < 16; ++c) {
        const uint4 x = got[r * 16 + c];
        if (x.x != h[r] || x.y != (uint32_t)c || x.z != 1u || x.w != 0xabcdu) ++bad;
      }
    std::printf("tma pull staging check: %llu bad vectors of %llu\n", (unsigned long long)bad, (unsigned long long)(req * 16));
  }
  run(3, 2, false, "tma pull 2 dir");
  run(3, 2, true, "tma pull 2 dir + copy");
  run(0, 2, true, "pull 2 dir + copy");
  run(1, 2, true, "push 2 dir + copy");
  return 0;
}
