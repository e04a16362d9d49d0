// Baseline cache rankings of the paper's Fig. 3 sweep, on the
// device: rank_degree, rank_halo_1hop, rank_wpr, rank_numpaths
// (/root/reference/proj/src/policies.cpp:57-132). Each computes its score
// vector on the device and orders the partition's remotes with the same
// order_remotes rule as vk_rank_by_scores (policies.cpp:20-34).
//
// Exactness: wPR and numpaths sum over in-neighbours in CSR order, one thread
// per row with round-to-nearest intrinsics (no FMA contraction), so every
// f64 score is bit-identical to the reference's sequential loops; wPR's
// dangling mass is a sequential sum over the (few) out-degree-0 vertices,
// done on the host in ascending id order exactly as the reference does.
#include <algorithm>
#include <cstring>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace vk {
namespace {

unsigned pgrid(std::uint64_t work, int device) {
  const std::uint64_t g = (work + 255) / 256;
  const std::uint64_t cap = (std::uint64_t)sm_count(device) * 16;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

// One BFS level of forward_reachable (policies.cpp:36-53): unseen out-
// neighbours of the current level join the next one.
__global__ void k_bfs_level(const std::uint64_t* __restrict__ off, const std::uint32_t* __restrict__ tgt,
                            const std::uint32_t* __restrict__ cur, std::uint32_t ncur, unsigned* __restrict__ seen,
                            std::uint32_t* __restrict__ next, unsigned* __restrict__ nnext) {
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t w0 = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) >> 5;
  const std::uint64_t nw = ((std::uint64_t)gridDim.x * blockDim.x) >> 5;
  for (std::uint64_t i = w0; i < ncur; i += nw) {
    const std::uint32_t v = cur[i];
    for (std::uint64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
      const std::uint32_t u = __ldg(tgt + e);
      if (!seen[u] && atomicExch(seen + u, 1u) == 0u) next[atomicAdd(nnext, 1u)] = u;
    }
  }
}

// rank_halo_1hop: remote out-neighbours of partition-k members score 1.
__global__ void k_halo(const std::uint64_t* __restrict__ off, const std::uint32_t* __restrict__ tgt,
                       const std::uint32_t* __restrict__ part_of, std::uint64_t n, std::uint32_t k,
                       double* __restrict__ score) {
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t w0 = (blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x) >> 5;
  const std::uint64_t nw = ((std::uint64_t)gridDim.x * blockDim.x) >> 5;
  for (std::uint64_t v = w0; v < n; v += nw) {
    if (part_of[v] != k) continue;
    for (std::uint64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
      const std::uint32_t u = __ldg(tgt + e);
      if (part_of[u] != k) score[u] = 1.0;
    }
  }
}

// One wPR power step (policies.cpp:104-113), row u: acc over in-neighbours
// in CSR order of rank[v] * (w / (w * deg v)), w = TransitionModel::weight.
__global__ void k_wpr_step(const std::uint64_t* __restrict__ roff, const std::uint32_t* __restrict__ rtgt,
                           const std::uint32_t* __restrict__ deg, std::uint64_t n, double f1,
                           const double* __restrict__ rank, const double* __restrict__ restart, double damping,
                           double dangling, double* __restrict__ next) {
  for (std::uint64_t u = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (std::uint64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (std::uint64_t e = roff[u]; e < roff[u + 1]; ++e) {
      const std::uint32_t v = __ldg(rtgt + e);
      const double d = (double)__ldg(deg + v);
      const double w = d <= f1 ? 1.0 : __ddiv_rn(f1, d);
      acc = __dadd_rn(acc, __dmul_rn(rank[v], __ddiv_rn(w, __dmul_rn(w, d))));
    }
    const double r = restart[u];
    next[u] = __dadd_rn(__dmul_rn(__dadd_rn(1.0, -damping), r), __dmul_rn(damping, __dadd_rn(acc, __dmul_rn(dangling, r))));
  }
}

// One numpaths hop (policies.cpp:122-131): next[u] = sum of count over
// in-neighbours (CSR order); scores += next.
__global__ void k_paths_step(const std::uint64_t* __restrict__ roff, const std::uint32_t* __restrict__ rtgt,
                             std::uint64_t n, const double* __restrict__ count, double* __restrict__ next,
                             double* __restrict__ scores) {
  for (std::uint64_t u = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (std::uint64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (std::uint64_t e = roff[u]; e < roff[u + 1]; ++e) acc = __dadd_rn(acc, count[__ldg(rtgt + e)]);
    next[u] = acc;
    scores[u] = __dadd_rn(scores[u], acc);
  }
}

__global__ void k_gather_f64(const double* __restrict__ src, const std::uint32_t* __restrict__ idx, std::uint64_t c,
                             double* __restrict__ out) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < c;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

std::vector<std::uint32_t> train_members(std::uint64_t n, const std::uint8_t* roles, const std::uint32_t* part_of,
                                         std::uint32_t k) {  // graph.cpp:106-111
  std::vector<std::uint32_t> t;
  for (std::uint64_t v = 0; v < n; ++v)
    if (part_of[v] == k && roles[v] == 0) t.push_back((std::uint32_t)v);
  return t;
}

void check_common(vk_graph g, const std::uint32_t* part_of, std::uint32_t K, std::uint32_t k, const void* order,
                  const void* score, const void* count) {
  if (!g || !part_of || !order || !score || !count) raise(VK_ERR_PARAMETER, "null argument");
  if (K == 0 || k >= K) raise(VK_ERR_PARAMETER, "partition index out of range");
  for (std::uint64_t v = 0; v < g->n; ++v)
    if (part_of[v] >= K) raise(VK_ERR_FORMAT, "partition label out of range");
}

void order_by(vk_graph g, const std::uint32_t* part_of, std::uint32_t k, const std::vector<double>& scores,
              std::uint32_t* order, double* score, std::uint64_t* count) {
  if (int e = vk_rank_by_scores(g->device, g->n, part_of, k, scores.data(), scores.size(), order, score, count))
    raise(e, vk_last_error());
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" {

int vk_rank_degree(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                   uint32_t L, uint32_t* order, double* score, uint64_t* count) {
  return guard([&] {
    check_common(g, part_of, K, k, order, score, count);
    if (!roles) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(g->device);
    const std::uint64_t n = g->n;
    const auto train = train_members(n, roles, part_of, k);
    DevBuf seen(n * 4), cur(n * 4), nxt(n * 4), cnt(4);
    std::uint32_t ncur = (std::uint32_t)train.size();
    if (ncur) VK_CUDA(cudaMemcpy(cur.p, train.data(), ncur * 4, cudaMemcpyHostToDevice));
    std::vector<unsigned> seen_h(n, 0);  // the sources are seen (policies.cpp:40)
    for (std::uint32_t v : train) seen_h[v] = 1;
    VK_CUDA(cudaMemcpy(seen.p, seen_h.data(), n * 4, cudaMemcpyHostToDevice));
    for (std::uint32_t h = 0; h < L && ncur; ++h) {
      VK_CUDA(cudaMemset(cnt.p, 0, 4));
      k_bfs_level<<<pgrid((std::uint64_t)ncur * 32, g->device), 256>>>(
          g->d_off(), g->d_tgt(), cur.as<std::uint32_t>(), ncur, seen.as<unsigned>(), nxt.as<std::uint32_t>(),
          cnt.as<unsigned>());
      count_launch();
      VK_LAUNCH_CHECK();
      VK_CUDA(cudaMemcpy(&ncur, cnt.p, 4, cudaMemcpyDeviceToHost));
      std::swap(cur, nxt);
    }
    VK_CUDA(cudaMemcpy(seen_h.data(), seen.p, n * 4, cudaMemcpyDeviceToHost));
    std::vector<std::uint32_t> deg(n);
    VK_CUDA(cudaMemcpy(deg.data(), g->out_deg.p, n * 4, cudaMemcpyDeviceToHost));
    // order_remotes with the reachability tier first (policies.cpp:62-64):
    // reachable vertices sort as deg + 1 > 0, unreachable ones as 0
    std::vector<double> comp(n, 0.0);
    for (std::uint64_t v = 0; v < n; ++v)
      if (seen_h[v]) comp[v] = (double)deg[v] + 1.0;
    order_by(g, part_of, k, comp, order, score, count);
    for (std::uint64_t i = 0; i < *count; ++i) score[i] = seen_h[order[i]] ? (double)deg[order[i]] : 0.0;
  });
}

int vk_rank_halo_1hop(vk_graph g, const uint32_t* part_of, uint32_t K, uint32_t k, uint32_t* order, double* score,
                      uint64_t* count, double* effective_alpha) {
  return guard([&] {
    check_common(g, part_of, K, k, order, score, count);
    DeviceGuard dg(g->device);
    const std::uint64_t n = g->n;
    DevBuf dpart(n * 4), dsc(n * 8);
    VK_CUDA(cudaMemcpy(dpart.p, part_of, n * 4, cudaMemcpyHostToDevice));
    VK_CUDA(cudaMemset(dsc.p, 0, n * 8));
    k_halo<<<pgrid(n * 32, g->device), 256>>>(g->d_off(), g->d_tgt(), dpart.as<std::uint32_t>(), n, k,
                                              dsc.as<double>());
    count_launch();
    VK_LAUNCH_CHECK();
    std::vector<double> sc(n);
    VK_CUDA(cudaMemcpy(sc.data(), dsc.p, n * 8, cudaMemcpyDeviceToHost));
    std::uint64_t halo = 0;
    for (double x : sc) halo += x != 0.0;
    order_by(g, part_of, k, sc, order, score, count);
    if (effective_alpha)  // policies.cpp:77-78
      *effective_alpha = (double)halo * (double)K / (double)n;
  });
}

int vk_rank_wpr(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                uint32_t hop1_fanout, uint32_t iters, double damping, uint32_t* order, double* score,
                uint64_t* count) {
  return guard([&] {
    check_common(g, part_of, K, k, order, score, count);
    if (!roles) raise(VK_ERR_PARAMETER, "null argument");
    if (iters < 1) raise(VK_ERR_PARAMETER, "wPR needs at least one iteration");  // policies.cpp:84
    if (hop1_fanout < 1) raise(VK_ERR_PARAMETER, "each fanout must be >= 1");
    DeviceGuard dg(g->device);
    const std::uint64_t n = g->n;
    const auto train = train_members(n, roles, part_of, k);
    if (train.empty()) raise(VK_ERR_SAMPLING, "partition has no train vertices");  // policies.cpp:87
    std::vector<double> restart(n, 0.0);
    const double e = 1.0 / (double)train.size();
    for (std::uint32_t v : train) restart[v] = e;
    std::vector<std::uint32_t> deg(n), dang;
    VK_CUDA(cudaMemcpy(deg.data(), g->out_deg.p, n * 4, cudaMemcpyDeviceToHost));
    for (std::uint64_t v = 0; v < n; ++v)
      if (deg[v] == 0) dang.push_back((std::uint32_t)v);
    DevBuf d_rs(n * 8), d_a(n * 8), d_b(n * 8), d_dang(std::max<std::size_t>(1, dang.size() * 4)),
        d_dv(std::max<std::size_t>(1, dang.size() * 8));
    VK_CUDA(cudaMemcpy(d_rs.p, restart.data(), n * 8, cudaMemcpyHostToDevice));
    VK_CUDA(cudaMemcpy(d_a.p, restart.data(), n * 8, cudaMemcpyHostToDevice));
    if (!dang.empty()) VK_CUDA(cudaMemcpy(d_dang.p, dang.data(), dang.size() * 4, cudaMemcpyHostToDevice));
    std::vector<double> dv(dang.size());
    for (std::uint32_t it = 0; it < iters; ++it) {
      double dangling = 0.0;  // ascending-id sequential sum (policies.cpp:101-103)
      if (!dang.empty()) {
        k_gather_f64<<<pgrid(dang.size(), g->device), 256>>>(d_a.as<double>(), d_dang.as<std::uint32_t>(),
                                                             dang.size(), d_dv.as<double>());
        count_launch();
        VK_CUDA(cudaMemcpy(dv.data(), d_dv.p, dang.size() * 8, cudaMemcpyDeviceToHost));
        for (double x : dv) dangling += x;
      }
      k_wpr_step<<<pgrid(n, g->device), 256>>>(g->rev_off, g->rev_tgt, g->out_deg.as<std::uint32_t>(), n,
                                               (double)hop1_fanout, d_a.as<double>(), d_rs.as<double>(), damping,
                                               dangling, d_b.as<double>());
      count_launch();
      VK_LAUNCH_CHECK();
      std::swap(d_a, d_b);
    }
    std::vector<double> rank(n);
    VK_CUDA(cudaMemcpy(rank.data(), d_a.p, n * 8, cudaMemcpyDeviceToHost));
    order_by(g, part_of, k, rank, order, score, count);
  });
}

int vk_rank_numpaths(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k, uint32_t L,
                     uint32_t* order, double* score, uint64_t* count) {
  return guard([&] {
    check_common(g, part_of, K, k, order, score, count);
    if (!roles) raise(VK_ERR_PARAMETER, "null argument");
    DeviceGuard dg(g->device);
    const std::uint64_t n = g->n;
    std::vector<double> c0(n, 0.0);
    for (std::uint32_t v : train_members(n, roles, part_of, k)) c0[v] = 1.0;
    DevBuf d_c(n * 8), d_n(n * 8), d_s(n * 8);
    VK_CUDA(cudaMemcpy(d_c.p, c0.data(), n * 8, cudaMemcpyHostToDevice));
    VK_CUDA(cudaMemset(d_s.p, 0, n * 8));
    for (std::uint32_t h = 0; h < L; ++h) {
      k_paths_step<<<pgrid(n, g->device), 256>>>(g->rev_off, g->rev_tgt, n, d_c.as<double>(), d_n.as<double>(),
                                                 d_s.as<double>());
      count_launch();
      VK_LAUNCH_CHECK();
      std::swap(d_c, d_n);
    }
    std::vector<double> sc(n);
    VK_CUDA(cudaMemcpy(sc.data(), d_s.p, n * 8, cudaMemcpyDeviceToHost));
    order_by(g, part_of, k, sc, order, score, count);
  });
}

}  // extern "C"
