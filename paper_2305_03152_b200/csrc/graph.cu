// Device-resident CSR graph: upload, on-device transpose (reverse CSR),
// invariant checks and the VCSR loader. Replaces vipkit::Graph +
// load_binary_csr (/root/reference/proj/include/vipkit/graph.hpp:20-46,117;
// src/graph.cpp:55-75, 565-598).
#include <cub/cub.cuh>

#include <cstring>
#include <fstream>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace vk {
namespace {

__global__ void k_out_degree(const std::uint64_t* __restrict__ off, std::uint64_t n,
                             std::uint32_t* __restrict__ deg, unsigned* __restrict__ max_deg) {
  std::uint32_t local_max = 0;
  for (std::uint64_t v = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t d = off[v + 1] - off[v];
    const std::uint32_t dd = d > 0xffffffffull ? 0xffffffffu : (std::uint32_t)d;
    deg[v] = dd;
    local_max = dd > local_max ? dd : local_max;
  }
  local_max = __reduce_max_sync(0xffffffffu, local_max);
  if ((threadIdx.x & 31) == 0) atomicMax(max_deg, local_max);
}

// check_invariants (graph.cpp:55-75): offsets non-decreasing, targets in
// range, no self-loops, strictly increasing per row. err bit codes:
// 1 offsets decrease, 2 target out of range, 4 self loop, 8 not increasing.
__global__ void k_check_rows(const std::uint64_t* __restrict__ off, const std::uint32_t* __restrict__ tgt,
                             std::uint64_t n, unsigned* __restrict__ err) {
  for (std::uint64_t v = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t a = off[v], b = off[v + 1];
    unsigned e = 0;
    if (a > b) {
      e |= 1;
    } else {
      for (std::uint64_t i = a; i < b; ++i) {
        const std::uint32_t t = tgt[i];
        if (t >= n) e |= 2;
        if (t == v) e |= 4;
        if (i > a && tgt[i - 1] >= t) e |= 8;
      }
    }
    if (e) atomicOr(err, e);
  }
}

// Reverse CSR by a key sort: key = (target << 32) | source, so each reverse
// row comes out sorted by source id (the order graph.cpp:593-595 produces).
__global__ void k_edge_keys(const std::uint64_t* __restrict__ off, std::uint64_t n,
                            const std::uint32_t* __restrict__ tgt, std::uint64_t* __restrict__ keys) {
  for (std::uint64_t u = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (std::uint64_t)gridDim.x * blockDim.x)
    for (std::uint64_t i = off[u]; i < off[u + 1]; ++i) keys[i] = ((std::uint64_t)tgt[i] << 32) | u;
}

__global__ void k_split_keys(const std::uint64_t* __restrict__ keys, std::uint64_t m,
                             std::uint32_t* __restrict__ rtgt, unsigned long long* __restrict__ counts) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint64_t k = keys[i];
    rtgt[i] = (std::uint32_t)k;
    atomicAdd(&counts[(k >> 32) + 1], 1ull);
  }
}

// apply_reorder (reorder.cpp:36-70): new row u is old row old_of_new[u] with
// every target mapped through new_of_old, emitted as sortable (u, t') keys.
__global__ void k_invert_perm(const std::uint32_t* __restrict__ old_of_new, std::uint64_t n,
                              std::uint32_t* __restrict__ new_of_old, unsigned* __restrict__ bad) {
  for (std::uint64_t u = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (std::uint64_t)gridDim.x * blockDim.x) {
    const std::uint32_t o = old_of_new[u];
    if (o >= n) {
      atomicOr(bad, 1u);
    } else if (atomicExch(new_of_old + o, (std::uint32_t)u) != 0xffffffffu) {
      atomicOr(bad, 2u);  // two new ids for one old vertex
    }
  }
}
__global__ void k_new_degrees(const std::uint32_t* __restrict__ old_of_new, const std::uint32_t* __restrict__ deg,
                              std::uint64_t n, std::uint64_t* __restrict__ new_off) {
  for (std::uint64_t u = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (std::uint64_t)gridDim.x * blockDim.x)
    new_off[u + 1] = deg[old_of_new[u]];
}
// warp per new row (power-law rows: lanes stride the row)
__global__ void k_relabel_rows(const std::uint64_t* __restrict__ off, const std::uint32_t* __restrict__ tgt,
                               const std::uint32_t* __restrict__ old_of_new,
                               const std::uint32_t* __restrict__ new_of_old, const std::uint64_t* __restrict__ new_off,
                               std::uint64_t n, std::uint64_t* __restrict__ keys) {
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t w0 = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) >> 5;
  const std::uint64_t nw = ((std::uint64_t)gridDim.x * blockDim.x) >> 5;
  for (std::uint64_t u = w0; u < n; u += nw) {
    const std::uint32_t o = old_of_new[u];
    const std::uint64_t b = off[o], e = off[o + 1], d = new_off[u];
    for (std::uint64_t i = b + lane; i < e; i += 32)
      keys[d + (i - b)] = (u << 32) | new_of_old[__ldg(tgt + i)];
  }
}
__global__ void k_low_words(const std::uint64_t* __restrict__ keys, std::uint64_t m, std::uint32_t* __restrict__ out) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    out[i] = (std::uint32_t)keys[i];
}

__global__ void k_compare(const std::uint64_t* __restrict__ a, const std::uint64_t* __restrict__ b,
                          std::uint64_t n64, const std::uint32_t* __restrict__ c,
                          const std::uint32_t* __restrict__ d, std::uint64_t n32, unsigned* __restrict__ diff) {
  bool any = false;
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < n64 || i < n32;
       i += (std::uint64_t)gridDim.x * blockDim.x) {
    if (i < n64 && a[i] != b[i]) any = true;
    if (i < n32 && c[i] != d[i]) any = true;
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(diff, 1u);
}

unsigned grid_for(std::uint64_t work, int device, unsigned block = 256) {
  const std::uint64_t g = (work + block - 1) / block;
  const std::uint64_t cap = (std::uint64_t)sm_count(device) * 16;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

void check_rows(vk_graph_s& g, const std::uint64_t* off, const std::uint32_t* tgt, const char* side) {
  DevBuf err(sizeof(unsigned));
  VK_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned), g.stream));
  if (g.n) {
    k_check_rows<<<grid_for(g.n, g.device), 256, 0, g.stream>>>(off, tgt, g.n, err.as<unsigned>());
    count_launch();
    VK_LAUNCH_CHECK();
  }
  unsigned h = 0;
  std::uint64_t ends[2] = {1, 1};
  VK_CUDA(cudaMemcpyAsync(&h, err.p, sizeof h, cudaMemcpyDeviceToHost, g.stream));
  VK_CUDA(cudaMemcpyAsync(&ends[0], off, 8, cudaMemcpyDeviceToHost, g.stream));
  VK_CUDA(cudaMemcpyAsync(&ends[1], off + g.n, 8, cudaMemcpyDeviceToHost, g.stream));
  VK_CUDA(cudaStreamSynchronize(g.stream));
  const std::string s(side);
  if (ends[0] != 0 || ends[1] != g.m) raise(VK_ERR_FORMAT, s + " offsets malformed");
  if (h & 1) raise(VK_ERR_FORMAT, s + " offsets decrease");
  if (h & 2) raise(VK_ERR_FORMAT, s + " target out of range");
  if (h & 4) raise(VK_ERR_FORMAT, "self-loop survived preprocessing");
  if (h & 8) raise(VK_ERR_FORMAT, s + " targets not strictly increasing");
}

// Reverse CSR on the device (graph.cpp:587-595 semantics).
void build_reverse(vk_graph_s& g) {
  const std::uint64_t n = g.n, m = g.m;
  g.rev_off_buf.alloc((n + 1) * 8);
  g.rev_tgt_buf.alloc(m ? m * 4 : 4);
  VK_CUDA(cudaMemsetAsync(g.rev_off_buf.p, 0, (n + 1) * 8, g.stream));
  if (m) {
    DevBuf keys(m * 8), keys2(m * 8);
    k_edge_keys<<<grid_for(n, g.device), 256, 0, g.stream>>>(g.d_off(), n, g.d_tgt(),
                                                             keys.as<std::uint64_t>());
    count_launch();
    VK_LAUNCH_CHECK();
    int end_bit = 32;
    while ((1ull << (end_bit - 32)) < n && end_bit < 64) ++end_bit;
    std::size_t tmp = 0;
    VK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.as<std::uint64_t>(),
                                           keys2.as<std::uint64_t>(), (std::int64_t)m, 0, end_bit,
                                           g.stream));
    DevBuf tbuf(tmp);
    VK_CUDA(cub::DeviceRadixSort::SortKeys(tbuf.p, tmp, keys.as<std::uint64_t>(),
                                           keys2.as<std::uint64_t>(), (std::int64_t)m, 0, end_bit,
                                           g.stream));
    count_launch(4);
    k_split_keys<<<grid_for(m, g.device), 256, 0, g.stream>>>(
        keys2.as<std::uint64_t>(), m, g.rev_tgt_buf.as<std::uint32_t>(),
        reinterpret_cast<unsigned long long*>(g.rev_off_buf.p));
    count_launch();
    VK_LAUNCH_CHECK();
    std::size_t tmp2 = 0;
    std::uint64_t* ro = g.rev_off_buf.as<std::uint64_t>();
    VK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp2, ro, ro, (std::int64_t)(n + 1), g.stream));
    DevBuf t2(tmp2);
    VK_CUDA(cub::DeviceScan::InclusiveSum(t2.p, tmp2, ro, ro, (std::int64_t)(n + 1), g.stream));
    count_launch();
    VK_CUDA(cudaStreamSynchronize(g.stream));
  }
  g.rev_off = g.rev_off_buf.as<std::uint64_t>();
  g.rev_tgt = g.rev_tgt_buf.as<std::uint32_t>();
}

bool reverse_equals_forward(vk_graph_s& g) {
  DevBuf diff(sizeof(unsigned));
  VK_CUDA(cudaMemsetAsync(diff.p, 0, sizeof(unsigned), g.stream));
  k_compare<<<grid_for(g.n + 1 > g.m ? g.n + 1 : g.m, g.device), 256, 0, g.stream>>>(
      g.d_off(), g.rev_off, g.n + 1, g.d_tgt(), g.rev_tgt, g.m, diff.as<unsigned>());
  count_launch();
  VK_LAUNCH_CHECK();
  unsigned h = 1;
  VK_CUDA(cudaMemcpyAsync(&h, diff.p, sizeof h, cudaMemcpyDeviceToHost, g.stream));
  VK_CUDA(cudaStreamSynchronize(g.stream));
  return h == 0;
}

void finish_graph(vk_graph_s& g, const std::uint64_t* rev_off_host, const std::uint32_t* rev_tgt_host,
                  std::uint32_t flags) {
  // forward out-degrees (TransitionModel::weight input, vip.hpp:22-26)
  g.out_deg.alloc(g.n ? g.n * 4 : 4);
  DevBuf mx(sizeof(unsigned));
  VK_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned), g.stream));
  if (g.n) {
    k_out_degree<<<grid_for(g.n, g.device), 256, 0, g.stream>>>(g.d_off(), g.n,
                                                                g.out_deg.as<std::uint32_t>(),
                                                                mx.as<unsigned>());
    count_launch();
    VK_LAUNCH_CHECK();
  }
  if (flags & VK_GRAPH_VALIDATE) check_rows(g, g.d_off(), g.d_tgt(), "forward");
  if (flags & VK_GRAPH_UNDIRECTED) {
    g.symmetric = true;
    g.rev_off = g.d_off();
    g.rev_tgt = g.d_tgt();
    if (flags & VK_GRAPH_VALIDATE) {
      build_reverse(g);
      if (!reverse_equals_forward(g)) raise(VK_ERR_FORMAT, "graph flagged undirected is not symmetric");
      g.rev_off_buf.release();
      g.rev_tgt_buf.release();
      g.rev_off = g.d_off();
      g.rev_tgt = g.d_tgt();
    }
  } else if (rev_off_host) {
    g.rev_off_buf.alloc((g.n + 1) * 8);
    g.rev_tgt_buf.alloc(g.m ? g.m * 4 : 4);
    VK_CUDA(cudaMemcpyAsync(g.rev_off_buf.p, rev_off_host, (g.n + 1) * 8, cudaMemcpyHostToDevice, g.stream));
    if (g.m)
      VK_CUDA(cudaMemcpyAsync(g.rev_tgt_buf.p, rev_tgt_host, g.m * 4, cudaMemcpyHostToDevice, g.stream));
    g.rev_off = g.rev_off_buf.as<std::uint64_t>();
    g.rev_tgt = g.rev_tgt_buf.as<std::uint32_t>();
    if (flags & VK_GRAPH_VALIDATE) check_rows(g, g.rev_off, g.rev_tgt, "reverse");
    g.symmetric = reverse_equals_forward(g);
    if (g.symmetric) {
      g.rev_off_buf.release();
      g.rev_tgt_buf.release();
      g.rev_off = g.d_off();
      g.rev_tgt = g.d_tgt();
    }
  } else {
    build_reverse(g);
    g.symmetric = reverse_equals_forward(g);
    if (g.symmetric) {
      g.rev_off_buf.release();
      g.rev_tgt_buf.release();
      g.rev_off = g.d_off();
      g.rev_tgt = g.d_tgt();
    }
  }
  unsigned h = 0;
  VK_CUDA(cudaMemcpyAsync(&h, mx.p, sizeof h, cudaMemcpyDeviceToHost, g.stream));
  VK_CUDA(cudaStreamSynchronize(g.stream));
  g.max_out_degree = h;
}

vk_graph_s* new_graph(int device, std::uint64_t n, std::uint64_t m) {
  if (n == 0 || n > (1ull << 32)) raise(VK_ERR_RANGE, "vertex count out of range: " + std::to_string(n));
  int ndev = 0;
  VK_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) raise(VK_ERR_CUDA, "no such CUDA device: " + std::to_string(device));
  auto* g = new vk_graph_s();
  g->device = device;
  g->n = n;
  g->m = m;
  VK_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  return g;
}

std::uint64_t get_u64_le(const unsigned char* b) {
  std::uint64_t x;
  std::memcpy(&x, b, 8);  // little-endian host (x86/arm64)
  return x;
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" {

int vk_graph_create(int device, uint64_t n, uint64_t m, const uint64_t* fwd_offsets,
                    const uint32_t* fwd_targets, const uint64_t* rev_offsets,
                    const uint32_t* rev_targets, uint32_t flags, vk_graph* out) {
  return guard([&] {
    if (!out || !fwd_offsets || (m && !fwd_targets)) raise(VK_ERR_PARAMETER, "null argument");
    if (fwd_offsets[0] != 0 || fwd_offsets[n] != m) raise(VK_ERR_FORMAT, "forward offsets malformed");
    if ((rev_offsets == nullptr) != (rev_targets == nullptr && m > 0) && m > 0)
      raise(VK_ERR_PARAMETER, "rev_offsets and rev_targets must both be given or both NULL");
    DeviceGuard dg(device);
    vk_graph_s* g = new_graph(device, n, m);
    try {
      g->fwd_off.alloc((n + 1) * 8);
      g->fwd_tgt.alloc(m ? m * 4 : 4);
      VK_CUDA(cudaMemcpyAsync(g->fwd_off.p, fwd_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, g->stream));
      if (m) VK_CUDA(cudaMemcpyAsync(g->fwd_tgt.p, fwd_targets, m * 4, cudaMemcpyHostToDevice, g->stream));
      finish_graph(*g, rev_offsets, rev_targets, flags);
    } catch (...) {
      vk_graph_destroy(g);
      throw;
    }
    *out = g;
  });
}

int vk_graph_apply_reorder(vk_graph src, const uint32_t* old_of_new, vk_graph* out) {
  return guard([&] {
    if (!src || !old_of_new || !out) raise(VK_ERR_PARAMETER, "null argument");
    vk_graph_s& g = *src;
    DeviceGuard dg(g.device);
    const std::uint64_t n = g.n, m = g.m;
    vk_graph_s* ng = new_graph(g.device, n, m);
    try {
      cudaStream_t st = ng->stream;
      VK_CUDA(cudaStreamSynchronize(g.stream));
      DevBuf oon(n * 4), noo(n * 4), bad(4);
      VK_CUDA(cudaMemcpyAsync(oon.p, old_of_new, n * 4, cudaMemcpyHostToDevice, st));
      VK_CUDA(cudaMemsetAsync(noo.p, 0xff, n * 4, st));
      VK_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
      k_invert_perm<<<grid_for(n, g.device), 256, 0, st>>>(oon.as<std::uint32_t>(), n, noo.as<std::uint32_t>(),
                                                          bad.as<unsigned>());
      count_launch();
      VK_LAUNCH_CHECK();
      unsigned hb = 0;
      VK_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, st));
      VK_CUDA(cudaStreamSynchronize(st));
      if (hb) raise(VK_ERR_SHAPE, "reorder map is not a permutation of the vertex ids");  // reorder.cpp:39
      // offsets: new row u has old row old_of_new[u]'s degree
      ng->fwd_off.alloc((n + 1) * 8);
      ng->fwd_tgt.alloc(m ? m * 4 : 4);
      std::uint64_t* no = ng->fwd_off.as<std::uint64_t>();
      VK_CUDA(cudaMemsetAsync(no, 0, 8, st));
      k_new_degrees<<<grid_for(n, g.device), 256, 0, st>>>(oon.as<std::uint32_t>(), g.out_deg.as<std::uint32_t>(),
                                                          n, no);
      count_launch();
      std::size_t tmp = 0;
      VK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, no, no, (std::int64_t)(n + 1), st));
      {
        DevBuf t(tmp);
        VK_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, no, no, (std::int64_t)(n + 1), st));
        count_launch();
        VK_CUDA(cudaStreamSynchronize(st));
      }
      if (m) {
        // relabelled rows as (u, t') keys; one radix sort orders every row
        // (std::sort per row, reorder.cpp:50) since rows are already grouped
        DevBuf keys(m * 8), keys2(m * 8);
        k_relabel_rows<<<grid_for(n * 32, g.device), 256, 0, st>>>(g.d_off(), g.d_tgt(), oon.as<std::uint32_t>(),
                                                                   noo.as<std::uint32_t>(), no, n,
                                                                   keys.as<std::uint64_t>());
        count_launch();
        VK_LAUNCH_CHECK();
        int end_bit = 32;
        while ((1ull << (end_bit - 32)) < n && end_bit < 64) ++end_bit;
        std::size_t t2 = 0;
        VK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t2, keys.as<std::uint64_t>(), keys2.as<std::uint64_t>(),
                                               (std::int64_t)m, 0, end_bit, st));
        DevBuf tb(t2);
        VK_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, t2, keys.as<std::uint64_t>(), keys2.as<std::uint64_t>(),
                                               (std::int64_t)m, 0, end_bit, st));
        count_launch(4);
        k_low_words<<<grid_for(m, g.device), 256, 0, st>>>(keys2.as<std::uint64_t>(), m,
                                                           ng->fwd_tgt.as<std::uint32_t>());
        count_launch();
        VK_LAUNCH_CHECK();
        VK_CUDA(cudaStreamSynchronize(st));
      }
      // a relabelling of a symmetric graph is symmetric (rev aliases fwd);
      // otherwise the reverse CSR is rebuilt on the device
      finish_graph(*ng, nullptr, nullptr, g.symmetric ? VK_GRAPH_UNDIRECTED : 0u);
    } catch (...) {
      vk_graph_destroy(ng);
      throw;
    }
    *out = ng;
  });
}

int vk_graph_load_vcsr(int device, const char* path, uint32_t flags, vk_graph* out) {
  return guard([&] {
    if (!out || !path) raise(VK_ERR_PARAMETER, "null argument");
    std::ifstream in(path, std::ios::binary);
    if (!in) raise(VK_ERR_IO, std::string("cannot open ") + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "VCSR", 4) != 0) raise(VK_ERR_FORMAT, std::string(path) + ": bad magic");
    unsigned char hdr[20];
    in.read(reinterpret_cast<char*>(hdr), 20);
    if (!in) raise(VK_ERR_IO, std::string(path) + ": truncated file");
    std::uint32_t version;
    std::memcpy(&version, hdr, 4);
    if (version != 1) raise(VK_ERR_FORMAT, std::string(path) + ": unsupported version " + std::to_string(version));
    const std::uint64_t n = get_u64_le(hdr + 4), m = get_u64_le(hdr + 12);
    if (n > (1ull << 32)) raise(VK_ERR_RANGE, std::string(path) + ": vertex count exceeds in-memory limit");
    std::vector<std::uint64_t> off(n + 1);
    in.read(reinterpret_cast<char*>(off.data()), (std::streamsize)((n + 1) * 8));
    std::vector<std::uint64_t> raw(m);
    in.read(reinterpret_cast<char*>(raw.data()), (std::streamsize)(m * 8));
    if (!in) raise(VK_ERR_IO, std::string(path) + ": truncated file");
    // u64 targets -> u32 in parallel, range-checked (graph.cpp:580-584)
    std::vector<std::uint32_t> tgt(m);
    const unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    std::atomic<bool> bad{false};
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const std::uint64_t lo = m * t / T, hi = m * (t + 1) / T;
        for (std::uint64_t i = lo; i < hi; ++i) {
          if (raw[i] >= n) bad = true;
          tgt[i] = (std::uint32_t)raw[i];
        }
      });
    for (auto& x : th) x.join();
    if (bad) raise(VK_ERR_FORMAT, std::string(path) + ": target id out of range");
    raw.clear();
    raw.shrink_to_fit();
    // load_binary_csr always validates (graph.cpp:596)
    const int rc = vk_graph_create(device, n, m, off.data(), tgt.data(), nullptr, nullptr,
                                   (flags | VK_GRAPH_VALIDATE) & ~VK_GRAPH_UNDIRECTED, out);
    if (rc != VK_OK) raise(rc, vk_last_error());
  });
}

int vk_graph_destroy(vk_graph g) {
  return guard([&] {
    if (!g) return;
    {
      DeviceGuard dg(g->device);
      if (g->stream) cudaStreamDestroy(g->stream);
      g->stream = nullptr;
    }
    delete g;
  });
}

int vk_graph_info(vk_graph g, uint64_t* n, uint64_t* m, int* symmetric, int* device) {
  return guard([&] {
    if (!g) raise(VK_ERR_PARAMETER, "null graph");
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (symmetric) *symmetric = g->symmetric ? 1 : 0;
    if (device) *device = g->device;
  });
}

int vk_graph_copy_forward(vk_graph g, uint64_t* fwd_offsets, uint32_t* fwd_targets) {
  return guard([&] {
    if (!g) raise(VK_ERR_PARAMETER, "null graph");
    DeviceGuard dg(g->device);
    if (fwd_offsets) VK_CUDA(cudaMemcpy(fwd_offsets, g->d_off(), (g->n + 1) * 8, cudaMemcpyDeviceToHost));
    if (fwd_targets && g->m) VK_CUDA(cudaMemcpy(fwd_targets, g->d_tgt(), g->m * 4, cudaMemcpyDeviceToHost));
  });
}

int vk_graph_copy_reverse(vk_graph g, uint64_t* rev_offsets, uint32_t* rev_targets) {
  return guard([&] {
    if (!g) raise(VK_ERR_PARAMETER, "null graph");
    DeviceGuard dg(g->device);
    if (rev_offsets) VK_CUDA(cudaMemcpy(rev_offsets, g->rev_off, (g->n + 1) * 8, cudaMemcpyDeviceToHost));
    if (rev_targets && g->m) VK_CUDA(cudaMemcpy(rev_targets, g->rev_tgt, g->m * 4, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
