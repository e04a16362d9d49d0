// Random 32 B-sector read throughput of HBM (the bound of the VIP gathers
// and the sampler's CSR reads): each thread reads `per` random 32 B records
// (index from a splitmix hash) from a `bytes` buffer and accumulates them.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull; x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull; x = (x ^ (x >> 27)) * 0x94d049bb133111ebull; return x ^ (x >> 31);
}
template <int REC>
__global__ void k(const uint4* __restrict__ buf, unsigned long long nrec, int per, unsigned long long seed, uint4* out) {
  const unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  uint4 acc = make_uint4(0,0,0,0);
  for (int i = 0; i < per; i += 4) {
    uint4 v[4][REC / 16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned long long r = mix(seed ^ (t * 4096 + i + u)) & (nrec - 1);
#pragma unroll
      for (int q = 0; q < REC / 16; ++q) v[u][q] = __ldg(buf + r * (REC / 16) + q);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < REC / 16; ++q) { acc.x ^= v[u][q].x; acc.y ^= v[u][q].y; acc.z ^= v[u][q].z; acc.w ^= v[u][q].w; }
  }
  if (acc.x == 0x12345678u) out[0] = acc;
}
int main() {
  const size_t bytes = 8ull << 30;
  uint4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  uint4* out; cudaMalloc(&out, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int per = 64; const int threads = 256; const int blocks = 148 * 64;
  for (int gran : {128, 64, 32}) {
  cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
  size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
  printf("L2 fetch granularity limit %d (reads back %zu)\n", gran, got);
  for (int rec : {32, 64, 128}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (rec == 32) k<32><<<blocks, threads>>>(buf, bytes / 32, per, rep, out);
      else if (rec == 64) k<64><<<blocks, threads>>>(buf, bytes / 64, per, rep, out);
      else k<128><<<blocks, threads>>>(buf, bytes / 128, per, rep, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double moved = (double)blocks * threads * per * rec;
      if (rep == 2) printf("record %3d B: %.1f GB/s useful (%.2f G records/s)\n", rec, moved / ms / 1e6, (double)blocks * threads * per / ms / 1e6);
    }
  }
  }
  return 0;
}
