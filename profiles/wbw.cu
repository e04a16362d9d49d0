// Streaming write-only and copy bandwidth of one B200 (the gather's traffic
// is 93 % writes): 16 B stores over a 24 GiB buffer, evict-first (.cs) and
// default policy, and a 16 B-load/16 B-store copy; persistent grid.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    uint4 v = MODE == 2 ? __ldg(src + i) : make_uint4((unsigned)i, 1, 2, 3);
    if (MODE == 0)
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else
      dst[i] = v;
  }
}
int main() {
  const size_t bytes = 12ull << 30, n = bytes / 16;
  uint4 *a, *b;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMemset(b, 1, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"write .cs", "write", "copy (read+write)"};
  for (int mode = 0; mode < 3; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 512>>>(a, b, n);
      else if (mode == 1) k<1><<<148 * 8, 512>>>(a, b, n);
      else k<2><<<148 * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double moved = mode == 2 ? 2.0 * bytes : (double)bytes;
      if (rep == 2) printf("%-18s %.1f GB/s\n", names[mode], moved / ms / 1e6);
    }
  return 0;
}
