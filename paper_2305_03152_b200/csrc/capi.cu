// C-ABI plumbing (errors, device helpers) and the host-side pieces of the
// path: epoch_minibatches (a single sequential Fisher-Yates stream per
// (epoch, partition) -- inherently serial, so it stays on the host and is
// overlapped with device work), the cache capacity rule, and the synthetic
// data generators used by bench.py.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"
#include "rng.cuh"

namespace vk {

std::atomic<std::uint64_t> g_launches{0};

namespace {
thread_local std::string t_err;
}

void set_last_error(const std::string& msg) { t_err = msg; }

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (device >= (int)cache.size()) cache.resize(device + 1, 0);
  if (cache[device] == 0) {
    int v = 0;
    VK_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    cache[device] = v;
  }
  return cache[device];
}

// The epoch shuffle of epoch_minibatches (sampling.cpp:54-63): stream
// (0xB1, epoch, k) folded from the global seed, Fisher-Yates from the back.
void epoch_shuffle(std::uint32_t* perm, std::uint64_t T, std::uint32_t k, std::uint64_t epoch,
                   std::uint64_t global_seed) {
  std::uint64_t h = global_seed;
  h = key_step(h, tag::minibatch_perm);
  h = key_step(h, epoch);
  h = key_step(h, k);
  Stream rng(h);
  for (std::uint64_t i = T; i > 1; --i) std::swap(perm[i - 1], perm[rng.next_below(i)]);
}

}  // namespace vk

using namespace vk;

extern "C" {

const char* vk_last_error(void) { return t_err.c_str(); }

const char* vk_status_name(int s) {
  switch (s) {
    case VK_OK: return "ok";
    case VK_ERR_PARSE: return "parse_error";
    case VK_ERR_RANGE: return "range_error";
    case VK_ERR_PARAMETER: return "parameter_error";
    case VK_ERR_FORMAT: return "format_error";
    case VK_ERR_PARTITION: return "partition_error";
    case VK_ERR_SAMPLING: return "sampling_error";
    case VK_ERR_CONFIG: return "config_error";
    case VK_ERR_SHAPE: return "shape_error";
    case VK_ERR_IO: return "io_error";
    case VK_ERR_CUDA: return "cuda_error";
    case VK_ERR_UNSUPPORTED: return "unsupported";
    default: return "internal_error";
  }
}

int vk_version(void) { return 100; }

uint64_t vk_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int vk_device_count(int* count) {
  return guard([&] {
    if (!count) raise(VK_ERR_PARAMETER, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    int ok = 0;
    for (int d = 0; d < n; ++d) {
      int major = 0;
      VK_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d));
      ok += (major == 10);
    }
    *count = ok;
  });
}

int vk_device_alloc(int device, size_t bytes, void** out) {
  return guard([&] {
    if (!out) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(device);
    VK_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  });
}

int vk_device_free(void* p) {
  return guard([&] { VK_CUDA(cudaFree(p)); });
}

int vk_memcpy(void* dst, const void* src, size_t bytes, int kind) {
  return guard([&] {
    // the library works on non-blocking streams, which a legacy-stream
    // cudaMemcpy does not order against: drain the device first
    VK_CUDA(cudaDeviceSynchronize());
    VK_CUDA(cudaMemcpy(dst, src, bytes, static_cast<cudaMemcpyKind>(kind)));
  });
}

int vk_stream_sync(vk_stream_t stream) {
  return guard([&] { VK_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
}

void vk_host_free(void* p) { std::free(p); }

// graph.cpp:106-111
int vk_train_members(uint64_t n, const uint8_t* roles, const uint32_t* part_of, uint32_t k, uint32_t* out,
                     uint64_t* out_count) {
  return guard([&] {
    if (!roles || !part_of || !out || !out_count) raise(VK_ERR_PARAMETER, "null argument");
    std::uint64_t T = 0;
    for (std::uint64_t v = 0; v < n; ++v)
      if (part_of[v] == k && roles[v] == 0) out[T++] = (std::uint32_t)v;
    *out_count = T;
  });
}

// sampling.cpp:54-63 over a precomputed train list
int vk_epoch_shuffle(const uint32_t* train, uint64_t count, uint32_t k, uint64_t epoch, uint64_t global_seed,
                     uint32_t* out) {
  return guard([&] {
    if ((!train && count) || !out) raise(VK_ERR_PARAMETER, "null argument");
    if (count == 0) raise(VK_ERR_SAMPLING, "partition " + std::to_string(k) + " has no train vertices");
    if (out != train) std::memcpy(out, train, count * 4);
    vk::epoch_shuffle(out, count, k, epoch, global_seed);
  });
}

// sampling.cpp:45-70 (+ train_members, graph.cpp:106-111).
int vk_epoch_minibatches(uint64_t n, const uint8_t* roles, const uint32_t* part_of, uint32_t k,
                         uint64_t batch_size, uint64_t epoch, uint64_t global_seed, const uint32_t* seed_keys,
                         uint32_t* out_perm, uint64_t* out_count) {
  return guard([&] {
    if (batch_size == 0) raise(VK_ERR_PARAMETER, "batch size must be >= 1");
    if (!roles || !part_of || !out_perm || !out_count) raise(VK_ERR_PARAMETER, "null argument");
    std::uint64_t T = 0;
    for (std::uint64_t v = 0; v < n; ++v)
      if (part_of[v] == k && roles[v] == 0) out_perm[T++] = (std::uint32_t)v;
    if (T == 0) raise(VK_ERR_SAMPLING, "partition " + std::to_string(k) + " has no train vertices");
    if (seed_keys)
      std::stable_sort(out_perm, out_perm + T,
                       [&](std::uint32_t a, std::uint32_t c) { return seed_keys[a] < seed_keys[c]; });
    vk::epoch_shuffle(out_perm, T, k, epoch, global_seed);
    *out_count = T;
  });
}

int vk_cache_capacity(double alpha, uint64_t n, uint32_t K, uint64_t* capacity) {
  return guard([&] {
    // policies.cpp:150-156
    if (!capacity) raise(VK_ERR_PARAMETER, "null argument");
    if (alpha < 0) raise(VK_ERR_PARAMETER, "replication factor must be >= 0");
    if (K == 0) raise(VK_ERR_PARAMETER, "need at least one ranking");
    *capacity = (std::uint64_t)std::floor(alpha * (double)n / (double)K + 1e-9);
  });
}

// make_roles (graph.cpp:247-268).
int vk_synth_roles(uint64_t n, double train, double valid, double test, uint64_t seed, uint8_t* roles) {
  return guard([&] {
    if (!roles) raise(VK_ERR_PARAMETER, "null argument");
    if (train < 0 || valid < 0 || test < 0 || train + valid + test > 1.0 + 1e-12)
      raise(VK_ERR_PARAMETER, "role fractions must be non-negative and sum to <= 1");
    std::vector<std::uint32_t> order(n);
    for (std::uint64_t i = 0; i < n; ++i) order[i] = (std::uint32_t)i;
    Stream rng(key_step(seed, tag::roles));
    for (std::uint64_t i = n; i > 1; --i) std::swap(order[i - 1], order[rng.next_below(i)]);
    std::memset(roles, 3, n);
    const auto t = (std::uint64_t)(train * (double)n);
    const auto va = (std::uint64_t)(valid * (double)n);
    const auto te = (std::uint64_t)(test * (double)n);
    std::uint64_t i = 0;
    for (std::uint64_t j = 0; j < t && i < n; ++j, ++i) roles[order[i]] = 0;
    for (std::uint64_t j = 0; j < va && i < n; ++j, ++i) roles[order[i]] = 1;
    for (std::uint64_t j = 0; j < te && i < n; ++j, ++i) roles[order[i]] = 2;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Community-structured power-law generator.
//
// Vertices are placed by a seeded permutation (ids carry no structure, like
// the reference PA generator's relabel, graph.cpp:195-201) into C balanced
// communities. Each vertex u emits d stubs; stub (u, j) draws from its own
// stream key (0xA1, 3, u, j): with probability p_in the target community is
// u's own, else uniform; the target is the community member of popularity
// rank floor(size * U^2) (a power-law in-degree, P(rank <= x) = sqrt(x/size)).
// Stubs are symmetrised, self-loops dropped, rows sorted and deduplicated
// (the Graph::from_edges canonical form, graph.cpp:33-53). Deterministic for
// any thread count: rows are sorted after the parallel fill.
namespace {

struct Perm {
  std::vector<std::uint32_t> rank_to_vertex, vertex_to_rank;
};

Perm make_perm(std::uint64_t n, std::uint64_t seed) {
  Perm p;
  p.rank_to_vertex.resize(n);
  for (std::uint64_t i = 0; i < n; ++i) p.rank_to_vertex[i] = (std::uint32_t)i;
  Stream rng(key_step(key_step(seed, 0xA1), 4));
  for (std::uint64_t i = n; i > 1; --i) std::swap(p.rank_to_vertex[i - 1], p.rank_to_vertex[rng.next_below(i)]);
  p.vertex_to_rank.resize(n);
  for (std::uint64_t i = 0; i < n; ++i) p.vertex_to_rank[p.rank_to_vertex[i]] = (std::uint32_t)i;
  return p;
}

template <class F>
void parallel_rows(unsigned T, std::uint64_t n, F&& fn) {
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      const std::uint64_t lo = n * t / T, hi = n * (t + 1) / T;
      fn(lo, hi);
    });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" int vk_synth_community_powerlaw(uint64_t n, uint64_t d, uint32_t communities, double p_in,
                                           uint64_t seed, unsigned threads, uint64_t** offsets,
                                           uint32_t** targets, uint64_t* m_out, uint32_t* labels) {
  return vk_synth_community_powerlaw_skew(n, d, communities, p_in, 2.0, seed, threads, offsets, targets, m_out,
                                          labels);
}

extern "C" int vk_synth_community_powerlaw_skew(uint64_t n, uint64_t d, uint32_t communities, double p_in,
                                                double skew, uint64_t seed, unsigned threads, uint64_t** offsets,
                                                uint32_t** targets, uint64_t* m_out, uint32_t* labels) {
  return guard([&] {
    if (!(skew >= 1.0 && skew <= 64.0)) raise(VK_ERR_PARAMETER, "skew must lie in [1, 64]");
    if (!offsets || !targets || !m_out) raise(VK_ERR_PARAMETER, "null argument");
    if (n < 2 || n > (1ull << 32)) raise(VK_ERR_RANGE, "vertex count out of range");
    if (d < 1) raise(VK_ERR_PARAMETER, "edges-per-vertex must be >= 1");
    if (communities < 1 || communities > n) raise(VK_ERR_PARAMETER, "bad community count");
    if (!(p_in >= 0.0 && p_in <= 1.0)) raise(VK_ERR_PARAMETER, "p_in must lie in [0,1]");
    const unsigned T = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
    const Perm perm = make_perm(n, seed);
    const std::uint32_t C = communities;
    auto cstart = [&](std::uint32_t c) { return (std::uint64_t)c * n / C; };
    auto comm_of_rank = [&](std::uint64_t r) {
      std::uint32_t c = (std::uint32_t)((r * C) / n);
      while (c + 1 < C && cstart(c + 1) <= r) ++c;
      while (cstart(c) > r) --c;
      return c;
    };
    if (labels)
      for (std::uint64_t v = 0; v < n; ++v) labels[v] = comm_of_rank(perm.vertex_to_rank[v]);
    const std::uint64_t base_key = key_step(key_step(seed, 0xA1), 3);
    auto stub = [&](std::uint64_t u, std::uint64_t j) -> std::uint32_t {
      Stream s(key_step(key_step(base_key, u), j));
      const std::uint32_t cu = comm_of_rank(perm.vertex_to_rank[u]);
      const double a = (double)(s.next_u64() >> 11) * 0x1.0p-53;
      const std::uint32_t c = a < p_in ? cu : (std::uint32_t)s.next_below(C);
      const std::uint64_t lo = cstart(c), size = cstart(c + 1) - lo;
      const double x = (double)(s.next_u64() >> 11) * 0x1.0p-53;
      std::uint64_t r = (std::uint64_t)((double)size * (skew == 2.0 ? x * x : std::pow(x, skew)));
      if (r >= size) r = size - 1;
      return perm.rank_to_vertex[lo + r];
    };
    // pass 1: degrees of the symmetrised multigraph
    std::vector<std::atomic<std::uint32_t>> deg(n);
    for (auto& x : deg) x.store(0, std::memory_order_relaxed);
    parallel_rows(T, n, [&](std::uint64_t lo, std::uint64_t hi) {
      for (std::uint64_t u = lo; u < hi; ++u)
        for (std::uint64_t j = 0; j < d; ++j) {
          const std::uint32_t t = stub(u, j);
          if (t == u) continue;
          deg[u].fetch_add(1, std::memory_order_relaxed);
          deg[t].fetch_add(1, std::memory_order_relaxed);
        }
    });
    std::vector<std::uint64_t> off(n + 1, 0);
    for (std::uint64_t v = 0; v < n; ++v) off[v + 1] = off[v] + deg[v].load(std::memory_order_relaxed);
    const std::uint64_t raw = off[n];
    std::vector<std::uint32_t> slots(raw);
    std::vector<std::atomic<std::uint64_t>> cur(n);
    for (std::uint64_t v = 0; v < n; ++v) cur[v].store(off[v], std::memory_order_relaxed);
    // pass 2: regenerate the same stubs and fill both directions
    parallel_rows(T, n, [&](std::uint64_t lo, std::uint64_t hi) {
      for (std::uint64_t u = lo; u < hi; ++u)
        for (std::uint64_t j = 0; j < d; ++j) {
          const std::uint32_t t = stub(u, j);
          if (t == u) continue;
          slots[cur[u].fetch_add(1, std::memory_order_relaxed)] = t;
          slots[cur[t].fetch_add(1, std::memory_order_relaxed)] = (std::uint32_t)u;
        }
    });
    // sort + dedup every row
    std::vector<std::uint64_t> newdeg(n);
    parallel_rows(T, n, [&](std::uint64_t lo, std::uint64_t hi) {
      for (std::uint64_t v = lo; v < hi; ++v) {
        auto* a = slots.data() + off[v];
        auto* b = slots.data() + off[v + 1];
        std::sort(a, b);
        newdeg[v] = (std::uint64_t)(std::unique(a, b) - a);
      }
    });
    auto* o = static_cast<std::uint64_t*>(std::malloc((n + 1) * 8));
    if (!o) raise(VK_ERR_INTERNAL, "host allocation failed");
    o[0] = 0;
    for (std::uint64_t v = 0; v < n; ++v) o[v + 1] = o[v] + newdeg[v];
    const std::uint64_t m = o[n];
    auto* t = static_cast<std::uint32_t*>(std::malloc(std::max<std::uint64_t>(m, 1) * 4));
    if (!t) {
      std::free(o);
      raise(VK_ERR_INTERNAL, "host allocation failed");
    }
    parallel_rows(T, n, [&](std::uint64_t lo, std::uint64_t hi) {
      for (std::uint64_t v = lo; v < hi; ++v) std::memcpy(t + o[v], slots.data() + off[v], newdeg[v] * 4);
    });
    *offsets = o;
    *targets = t;
    *m_out = m;
  });
}
