// simulate (commsim.cpp:77-127) and the alpha axis of sweep
// (commsim.cpp:140-259) on the device -- SURVEY §8f row F1.
//
// The reference expands every minibatch of every partition for E epochs
// (for_each_expansion, commsim.cpp:38-52: epoch-major, then partition, then
// batch index) and classifies each distinct neighbourhood vertex of the
// minibatch of partition k as local (part_of[v] == k), cache hit
// (CachePlan::is_cached(k, v)) or remote miss (classify, commsim.cpp:61-73),
// summing per (epoch, partition) cell. Expansion depends only on the seeds, so
// here the minibatches stream through the batched device sampler in waves and
// one classification pass scores them against several cache plans at once:
// plan a caches the first takes[a][k] ids of partition k's cached list (the
// ranking prefixes build_cache produces, policies.cpp:149-163), so a vertex
// at list position p is a hit for every plan with takes > p.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "rng.cuh"

struct vk_sampler_s;
namespace vk {
void sampler_internal(vk_sampler_s* s, const std::uint32_t** all, std::uint64_t* all_stride,
                      const std::uint32_t** all_count, std::uint32_t* nmb, const std::uint32_t** partitions,
                      vk_graph_s** g, cudaStream_t* last_stream);
}  // namespace vk

namespace vk {
namespace {

constexpr std::uint32_t kMaxPlans = 32;

unsigned fill_grid(std::uint64_t work, int device) {
  const std::uint64_t g = (work + 255) / 256;
  const std::uint64_t cap = (std::uint64_t)sm_count(device) * 16;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

__global__ void k_fill_positions(const std::uint32_t* __restrict__ ids, std::uint64_t count,
                                 std::uint32_t* __restrict__ pos) {
  for (std::uint64_t i = blockIdx.x * (std::uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (std::uint64_t)gridDim.x * blockDim.x)
    pos[ids[i]] = (std::uint32_t)i;
}

// One (chunk, minibatch) CTA: per vertex of all_vertices, local / per-plan
// hit counts, reduced in shared memory and added to the minibatch's cell.
__global__ void __launch_bounds__(256) k_classify_plans(const std::uint32_t* __restrict__ all, std::uint64_t stride,
                                                        const std::uint32_t* __restrict__ count,
                                                        const std::uint32_t* __restrict__ cell_of,
                                                        const std::uint32_t* __restrict__ part_of,
                                                        const std::uint32_t* __restrict__ pos, std::uint64_t n,
                                                        const std::uint64_t* __restrict__ takes, std::uint32_t K,
                                                        std::uint32_t A, std::uint64_t cells_per_plan,
                                                        unsigned long long* __restrict__ cells,
                                                        unsigned long long* __restrict__ batch_cnt,
                                                        std::uint64_t batch_base,
                                                        const std::uint32_t* __restrict__ gpu_pos,
                                                        const std::uint64_t* __restrict__ gpu_cut) {
  __shared__ unsigned long long s_cnt[3 + kMaxPlans];
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t cell = cell_of[mb];
  const std::uint32_t k = cell % K;
  for (std::uint32_t i = threadIdx.x; i < 3 + A; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  std::uint64_t tk[kMaxPlans];
#pragma unroll
  for (std::uint32_t a = 0; a < kMaxPlans; ++a) tk[a] = a < A ? takes[a * K + k] : 0;
  unsigned long long local = 0, remote = 0, gpu_local = 0;
  const std::uint32_t* gp = gpu_pos ? gpu_pos + (std::uint64_t)k * n : nullptr;
  const std::uint64_t cut = gpu_pos ? gpu_cut[k] : 0;
  unsigned hits[kMaxPlans];
#pragma unroll
  for (std::uint32_t a = 0; a < kMaxPlans; ++a) hits[a] = 0;
  const std::uint32_t c = count[mb];
  const std::uint32_t* av = all + mb * stride;
  const std::uint32_t* pk = pos + (std::uint64_t)k * n;
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < c; r += gridDim.x * blockDim.x) {
    const std::uint32_t v = __ldg(av + r);
    if (__ldg(part_of + v) == k) {
      ++local;
      if (gp && __ldg(gp + v) < cut) ++gpu_local;  // SimulateOptions GPU-prefix split
    } else {
      ++remote;
      const std::uint32_t p = __ldg(pk + v);
#pragma unroll
      for (std::uint32_t a = 0; a < kMaxPlans; ++a) hits[a] += (a < A && p < tk[a]) ? 1u : 0u;
    }
  }
  // warp reduction, then one shared atomic per warp and counter
  auto wsum = [](unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  local = wsum(local);
  remote = wsum(remote);
  gpu_local = wsum(gpu_local);
  const bool lead = (threadIdx.x & 31) == 0;
  if (lead) {
    atomicAdd(&s_cnt[0], local);
    atomicAdd(&s_cnt[1], remote);
    atomicAdd(&s_cnt[2], gpu_local);
  }
#pragma unroll
  for (std::uint32_t a = 0; a < kMaxPlans; ++a) {
    if (a < A) {
      const unsigned long long h = wsum(hits[a]);
      if (lead) atomicAdd(&s_cnt[3 + a], h);
    }
  }
  __syncthreads();
  if (threadIdx.x < A) {
    const std::uint32_t a = threadIdx.x;
    unsigned long long* cl = cells + a * cells_per_plan + (std::uint64_t)cell * 3;
    const unsigned long long h = s_cnt[3 + a];
    if (s_cnt[0]) atomicAdd(cl + 0, s_cnt[0]);
    if (h) atomicAdd(cl + 1, h);
    if (s_cnt[1] - h) atomicAdd(cl + 2, s_cnt[1] - h);
  }
  if (batch_cnt && threadIdx.x == 0) {  // per-minibatch rows of plan 0: local, gpu local, cache, miss
    unsigned long long* bc = batch_cnt + (batch_base + mb) * 4;
    atomicAdd(bc + 0, s_cnt[0]);
    atomicAdd(bc + 1, s_cnt[2]);
    atomicAdd(bc + 2, s_cnt[3]);
    atomicAdd(bc + 3, s_cnt[1] - s_cnt[3]);
  }
}

// empirical_vip's histogram: one count per distinct neighbourhood vertex of
// every minibatch of the wave.
__global__ void __launch_bounds__(256) k_histogram(const std::uint32_t* __restrict__ all, std::uint64_t stride,
                                                   const std::uint32_t* __restrict__ count,
                                                   unsigned* __restrict__ hits) {
  const std::uint32_t mb = blockIdx.y;
  const std::uint32_t c = count[mb];
  const std::uint32_t* av = all + mb * stride;
  for (std::uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < c; r += gridDim.x * blockDim.x)
    atomicAdd(hits + __ldg(av + r), 1u);
}

// for_each_expansion (commsim.cpp:38-52) over the device sampler: the
// minibatches of epochs x `parts` in the reference's order (epoch-major, then
// partition, then batch index) go through the sampler in waves of M; after
// each wave on_wave(all, stride, count, nmb, cells_of_wave, stream) launches
// the consumer on the sampler's stream. cells_of_wave[i] = e * K + k of
// minibatch i (host array, valid during the call). Returns the minibatch count.
template <class OnWave>
std::uint64_t stream_expansions(vk_graph g, const std::uint8_t* roles, const std::uint32_t* part_of,
                                std::uint32_t K, const std::vector<std::uint32_t>& parts,
                                const std::uint32_t* fanouts, std::uint32_t num_hops, std::uint64_t batch_size,
                                std::uint64_t epochs, std::uint64_t seed, const std::uint32_t* seed_keys,
                                std::uint32_t M, OnWave&& on_wave) {
  if (num_hops == 0 || num_hops > VK_MAX_HOPS) raise(VK_ERR_PARAMETER, "1..VK_MAX_HOPS hops");
  vk_sampler_config cfg{};
  cfg.num_hops = num_hops;
  for (std::uint32_t h = 0; h < num_hops; ++h) cfg.fanouts[h] = fanouts[h];
  cfg.batch_size = batch_size;
  cfg.max_minibatches = M;
  cfg.global_seed = seed;
  vk_sampler sampler = nullptr;
  if (int e = vk_sampler_create(g, &cfg, &sampler)) raise(e, vk_last_error());
  struct SamplerGuard {
    vk_sampler s;
    ~SamplerGuard() { vk_sampler_destroy(s); }
  } sg{sampler};
  if (seed_keys)
    if (int e = vk_sampler_set_seed_keys(sampler, seed_keys)) raise(e, vk_last_error());
  const std::uint64_t n = g->n;
  // train members of the partitions in ascending id order (train_members,
  // graph.cpp:106-111), gathered in one pass instead of one per (e, k)
  std::vector<int> want(K, 0);
  for (std::uint32_t k : parts) want[k] = 1;
  std::vector<std::vector<std::uint32_t>> members(K);
  for (std::uint64_t v = 0; v < n; ++v)
    if (roles[v] == 0 && want[part_of[v]]) members[part_of[v]].push_back((std::uint32_t)v);
  if (seed_keys)  // canonical order follows the replay keys (sampling.cpp:54-58)
    for (auto& mk : members)
      std::stable_sort(mk.begin(), mk.end(),
                       [&](std::uint32_t a, std::uint32_t c) { return seed_keys[a] < seed_keys[c]; });
  std::vector<std::uint32_t> perm, seeds, cell_of;
  std::vector<std::uint64_t> offs{0};
  std::vector<vk_batch_ref> refs;
  std::uint64_t total = 0;
  auto flush = [&] {
    if (refs.empty()) return;
    const std::uint32_t nmb = (std::uint32_t)refs.size();
    if (int e = vk_sampler_run(sampler, nmb, refs.data(), seeds.data(), offs.data(), 0, nullptr))
      raise(e, vk_last_error());
    const std::uint32_t *all, *count, *pt;
    std::uint64_t stride;
    std::uint32_t got;
    vk_graph_s* gg;
    cudaStream_t st;
    sampler_internal(sampler, &all, &stride, &count, &got, &pt, &gg, &st);
    on_wave(all, stride, count, nmb, cell_of.data(), st);
    total += nmb;
    seeds.clear();
    offs.assign(1, 0);
    refs.clear();
    cell_of.clear();
  };
  for (std::uint64_t e = 0; e < epochs; ++e)
    for (std::uint32_t k : parts) {
      if (members[k].empty())  // sampling.cpp:50-53
        raise(VK_ERR_SAMPLING, "partition " + std::to_string(k) + " has no train vertices");
      const std::uint64_t T = members[k].size();
      perm.assign(members[k].begin(), members[k].end());
      epoch_shuffle(perm.data(), T, k, e, seed);  // epoch_minibatches (sampling.cpp:45-70)
      for (std::uint64_t i = 0, bi = 0; i < T; i += batch_size, ++bi) {
        const std::uint64_t c = std::min<std::uint64_t>(batch_size, T - i);
        seeds.insert(seeds.end(), perm.begin() + i, perm.begin() + i + c);
        offs.push_back(seeds.size());
        refs.push_back(vk_batch_ref{e, bi, k, 0});
        cell_of.push_back((std::uint32_t)(e * K + k));
        if (refs.size() == M) flush();
      }
    }
  flush();
  VK_CUDA(cudaDeviceSynchronize());  // consumers ran on the sampler's (non-blocking) stream
  return total;
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" {

}  // extern "C"

namespace {
// vk_simulate / vk_simulate_batches: batch_rows (optional) receives one row
// per minibatch in for_each_expansion order {epoch, batch_index, partition,
// local - gpu, gpu, cache, miss} for plan 0 (commsim.cpp:104-118).
void simulate_core(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, const uint32_t* fanouts,
                   uint32_t num_hops, uint64_t batch_size, uint64_t epochs, uint64_t global_seed,
                   const uint32_t* seed_keys, const uint32_t* cached_ids, const uint64_t* cached_offsets,
                   const uint64_t* takes, uint32_t num_plans, uint32_t wave, uint64_t* cells,
                   const uint32_t* const* gpu_orderings, const uint64_t* gpu_ordering_sizes, double gamma,
                   uint64_t* batch_rows, uint64_t batch_rows_capacity, uint64_t* num_batches) {
  {
    if (!g || !roles || !part_of || !fanouts || !cached_offsets || !cells) raise(VK_ERR_PARAMETER, "null argument");
    if (K == 0) raise(VK_ERR_PARAMETER, "need at least one partition");
    if (batch_size == 0) raise(VK_ERR_PARAMETER, "batch size must be >= 1");  // sampling.cpp:50-53
    const std::uint32_t A = takes ? num_plans : 1u;
    if (A == 0 || A > kMaxPlans) raise(VK_ERR_PARAMETER, "between 1 and 32 cache plans per call");
    const std::uint64_t n = g->n;
    for (std::uint64_t v = 0; v < n; ++v)
      if (part_of[v] >= K) raise(VK_ERR_FORMAT, "partition label out of range");
    if (cached_offsets[0] != 0) raise(VK_ERR_SHAPE, "cached_offsets must start at 0");
    for (std::uint32_t k = 0; k < K; ++k)
      if (cached_offsets[k + 1] < cached_offsets[k]) raise(VK_ERR_SHAPE, "cached_offsets must be non-decreasing");
    const std::uint64_t ncached = cached_offsets[K];
    if (ncached && !cached_ids) raise(VK_ERR_PARAMETER, "null cached_ids");
    for (std::uint64_t i = 0; i < ncached; ++i)
      if (cached_ids[i] >= n) raise(VK_ERR_RANGE, "cached vertex id out of range");
    std::vector<std::uint64_t> tk(A * K);
    for (std::uint32_t a = 0; a < A; ++a)
      for (std::uint32_t k = 0; k < K; ++k) {
        const std::uint64_t len = cached_offsets[k + 1] - cached_offsets[k];
        tk[a * K + k] = takes ? takes[a * K + k] : len;
        if (tk[a * K + k] > len) raise(VK_ERR_SHAPE, "plan takes more ids than the cached list holds");
      }
    const std::uint32_t M = wave ? wave : 128u;
    DeviceGuard dg(g->device);
    const std::uint64_t ncell = epochs * K;
    DevBuf d_part, d_pos, d_takes, d_cells, d_cell_of, d_ids;
    d_part.alloc(n * 4);
    VK_CUDA(cudaMemcpy(d_part.p, part_of, n * 4, cudaMemcpyHostToDevice));
    d_pos.alloc((std::uint64_t)K * n * 4);
    VK_CUDA(cudaMemset(d_pos.p, 0xff, d_pos.bytes));
    if (ncached) {
      d_ids.alloc(ncached * 4);
      VK_CUDA(cudaMemcpy(d_ids.p, cached_ids, ncached * 4, cudaMemcpyHostToDevice));
      for (std::uint32_t k = 0; k < K; ++k) {
        const std::uint64_t c = cached_offsets[k + 1] - cached_offsets[k];
        if (c)
          k_fill_positions<<<fill_grid(c, g->device), 256>>>(d_ids.as<std::uint32_t>() + cached_offsets[k], c,
                                                           d_pos.as<std::uint32_t>() + (std::uint64_t)k * n);
      }
      VK_LAUNCH_CHECK();
    }
    d_takes.alloc(A * K * 8);
    VK_CUDA(cudaMemcpy(d_takes.p, tk.data(), A * K * 8, cudaMemcpyHostToDevice));
    d_cells.alloc(std::max<std::uint64_t>(1, A * ncell * 3 * 8));
    VK_CUDA(cudaMemset(d_cells.p, 0, d_cells.bytes));
    d_cell_of.alloc(2 * M * 4);  // double-buffered: the host fills wave i+1 while wave i runs
    // per-minibatch rows (SimulateOptions::batch_costs): the minibatch count
    // in for_each order, device counters [total][4], refs kept on the host
    DevBuf d_batch, d_gpu_pos, d_gpu_cut;
    std::vector<std::uint64_t> batch_refs;  // epoch, batch_index, partition
    if (batch_rows || num_batches) {
      std::vector<std::uint64_t> T(K, 0);
      for (std::uint64_t v = 0; v < n; ++v)
        if (roles[v] == 0) ++T[part_of[v]];
      std::uint64_t total = 0;
      for (std::uint32_t k = 0; k < K; ++k) total += (T[k] + batch_size - 1) / batch_size;
      total *= epochs;
      if (num_batches) *num_batches = total;
      if (batch_rows && batch_rows_capacity < total) raise(VK_ERR_SHAPE, "batch_rows capacity below the minibatch count");
      if (batch_rows) {
        d_batch.alloc(std::max<std::uint64_t>(1, total) * 4 * 8);
        VK_CUDA(cudaMemset(d_batch.p, 0, d_batch.bytes));
        batch_refs.reserve(total * 3);
        for (std::uint64_t e = 0; e < epochs; ++e)  // for_each_expansion order (commsim.cpp:45-52)
          for (std::uint32_t k = 0; k < K; ++k)
            for (std::uint64_t i = 0; i * batch_size < T[k]; ++i) {
              batch_refs.push_back(e);
              batch_refs.push_back(i);
              batch_refs.push_back(k);
            }
      }
    }
    if (batch_rows && gpu_orderings) {
      // gpu_threshold_pos / gpu_cut of commsim.cpp:91-102
      std::vector<std::uint32_t> pos((std::uint64_t)K * n, 0xffffffffu);
      std::vector<std::uint64_t> cut(K);
      for (std::uint32_t k = 0; k < K; ++k) {
        const std::uint64_t sz = gpu_ordering_sizes[k];
        for (std::uint64_t i = 0; i < sz; ++i) {
          const std::uint32_t v = gpu_orderings[k][i];
          if (v >= n) raise(VK_ERR_RANGE, "gpu ordering vertex out of range");
          pos[(std::uint64_t)k * n + v] = (std::uint32_t)std::min<std::uint64_t>(i, 0xfffffffeu);
        }
        cut[k] = (std::uint64_t)std::floor(gamma * (double)sz + 1e-9);
      }
      d_gpu_pos.alloc(pos.size() * 4);
      VK_CUDA(cudaMemcpy(d_gpu_pos.p, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice));
      d_gpu_cut.alloc(K * 8);
      VK_CUDA(cudaMemcpy(d_gpu_cut.p, cut.data(), K * 8, cudaMemcpyHostToDevice));
    }
    std::uint64_t batch_base = 0;
    VK_CUDA(cudaDeviceSynchronize());
    PinnedBuf cell_host;
    cell_host.ensure(2 * M * 4);
    cudaEvent_t copied[2] = {nullptr, nullptr};
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        for (int i = 0; i < 2; ++i)
          if (e[i]) cudaEventDestroy(e[i]);
      }
    } evg{copied};
    for (auto& ev : copied) VK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    int parity = 0;
    std::vector<std::uint32_t> parts(K);
    for (std::uint32_t k = 0; k < K; ++k) parts[k] = k;
    stream_expansions(g, roles, part_of, K, parts, fanouts, num_hops, batch_size, epochs, global_seed, seed_keys, M,
                      [&](const std::uint32_t* all, std::uint64_t stride, const std::uint32_t* count,
                          std::uint32_t nmb, const std::uint32_t* cell_of, cudaStream_t st) {
                        std::uint32_t* ch = cell_host.as<std::uint32_t>() + parity * M;
                        std::uint32_t* cd = d_cell_of.as<std::uint32_t>() + parity * M;
                        VK_CUDA(cudaEventSynchronize(copied[parity]));  // wave i-2 consumed this buffer
                        std::memcpy(ch, cell_of, nmb * 4);
                        VK_CUDA(cudaMemcpyAsync(cd, ch, nmb * 4, cudaMemcpyHostToDevice, st));
                        const unsigned gx = (unsigned)std::max<std::uint64_t>(
                            1, std::min<std::uint64_t>(ceil_div(stride, 256 * 8), 64));
                        k_classify_plans<<<dim3(gx, nmb), 256, 0, st>>>(
                            all, stride, count, cd, d_part.as<std::uint32_t>(), d_pos.as<std::uint32_t>(), n,
                            d_takes.as<std::uint64_t>(), K, A, ncell * 3, d_cells.as<unsigned long long>(),
                            d_batch.p ? d_batch.as<unsigned long long>() : nullptr, batch_base,
                            d_gpu_pos.p ? d_gpu_pos.as<std::uint32_t>() : nullptr,
                            d_gpu_cut.p ? d_gpu_cut.as<std::uint64_t>() : nullptr);
                        batch_base += nmb;
                        count_launch();
                        VK_LAUNCH_CHECK();
                        VK_CUDA(cudaEventRecord(copied[parity], st));
                        parity ^= 1;
                      });
    std::vector<unsigned long long> host(A * ncell * 3);
    if (!host.empty()) VK_CUDA(cudaMemcpy(host.data(), d_cells.p, host.size() * 8, cudaMemcpyDeviceToHost));
    for (std::size_t i = 0; i < host.size(); ++i) cells[i] = host[i];
    if (batch_rows) {
      std::vector<unsigned long long> bc(batch_base * 4);
      if (!bc.empty()) VK_CUDA(cudaMemcpy(bc.data(), d_batch.p, bc.size() * 8, cudaMemcpyDeviceToHost));
      for (std::uint64_t i = 0; i < batch_base; ++i) {
        std::uint64_t* r = batch_rows + i * 7;
        r[0] = batch_refs[3 * i];
        r[1] = batch_refs[3 * i + 1];
        r[2] = batch_refs[3 * i + 2];
        r[3] = bc[4 * i] - bc[4 * i + 1];
        r[4] = bc[4 * i + 1];
        r[5] = bc[4 * i + 2];
        r[6] = bc[4 * i + 3];
      }
    }
  }
}
}  // namespace

extern "C" {

int vk_simulate(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, const uint32_t* fanouts,
                uint32_t num_hops, uint64_t batch_size, uint64_t epochs, uint64_t global_seed,
                const uint32_t* seed_keys, const uint32_t* cached_ids, const uint64_t* cached_offsets, const uint64_t* takes,
                uint32_t num_plans, uint32_t wave, uint64_t* cells) {
  return guard([&] {
    simulate_core(g, roles, part_of, K, fanouts, num_hops, batch_size, epochs, global_seed, seed_keys, cached_ids,
                  cached_offsets, takes, num_plans, wave, cells, nullptr, nullptr, 0.0, nullptr, 0, nullptr);
  });
}

int vk_simulate_batches(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K,
                        const uint32_t* fanouts, uint32_t num_hops, uint64_t batch_size, uint64_t epochs,
                        uint64_t global_seed, const uint32_t* seed_keys, const uint32_t* cached_ids,
                        const uint64_t* cached_offsets, const uint32_t* const* gpu_orderings,
                        const uint64_t* gpu_ordering_sizes, double gamma, uint64_t* cells, uint64_t* batch_rows,
                        uint64_t batch_rows_capacity, uint64_t* num_batches) {
  return guard([&] {
    if (gpu_orderings && !gpu_ordering_sizes) raise(VK_ERR_PARAMETER, "null gpu ordering sizes");
    simulate_core(g, roles, part_of, K, fanouts, num_hops, batch_size, epochs, global_seed, seed_keys, cached_ids,
                  cached_offsets, nullptr, 1, 0, cells, gpu_orderings, gpu_ordering_sizes, gamma, batch_rows,
                  batch_rows_capacity, num_batches);
  });
}

// empirical_vip (vip.cpp:85-105): for S epochs, every minibatch of
// partition k under the derived seed (0xC1, rng.hpp:54), a histogram of
// all_vertices; freq[v] = hits[v] / batches.
int vk_empirical_vip(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, uint32_t k,
                     uint64_t batch_size, const uint32_t* fanouts, uint32_t num_hops, uint64_t epochs,
                     uint64_t global_seed, double* freq) {
  return guard([&] {
    if (!g || !roles || !part_of || !fanouts || !freq) raise(VK_ERR_PARAMETER, "null argument");
    if (epochs < 1) raise(VK_ERR_PARAMETER, "epoch count must be >= 1");  // vip.cpp:89
    if (batch_size == 0) raise(VK_ERR_PARAMETER, "batch size must be >= 1");
    if (K == 0 || k >= K) raise(VK_ERR_PARAMETER, "partition index out of range");
    const std::uint64_t n = g->n;
    for (std::uint64_t v = 0; v < n; ++v)
      if (part_of[v] >= K) raise(VK_ERR_FORMAT, "partition label out of range");
    for (std::uint32_t h = 0; h < num_hops; ++h)
      if (fanouts[h] < 1) raise(VK_ERR_PARAMETER, "each fanout must be >= 1");
    DeviceGuard dg(g->device);
    const std::uint64_t seed = mix64(global_seed ^ mix64(tag::empirical_vip));  // SeedSpec::derived
    DevBuf hits;
    hits.alloc(std::max<std::uint64_t>(1, n * 4));
    VK_CUDA(cudaMemset(hits.p, 0, hits.bytes));
    VK_CUDA(cudaDeviceSynchronize());
    const std::uint64_t batches = stream_expansions(
        g, roles, part_of, K, {k}, fanouts, num_hops, batch_size, epochs, seed, nullptr, 128u,
        [&](const std::uint32_t* all, std::uint64_t stride, const std::uint32_t* count, std::uint32_t nmb,
            const std::uint32_t*, cudaStream_t st) {
          const unsigned gx = (unsigned)std::max<std::uint64_t>(1, std::min<std::uint64_t>(ceil_div(stride, 256 * 8), 64));
          k_histogram<<<dim3(gx, nmb), 256, 0, st>>>(all, stride, count, hits.as<unsigned>());
          count_launch();
          VK_LAUNCH_CHECK();
        });
    std::vector<unsigned> h(n);
    if (n) VK_CUDA(cudaMemcpy(h.data(), hits.p, n * 4, cudaMemcpyDeviceToHost));
    for (std::uint64_t v = 0; v < n; ++v) freq[v] = static_cast<double>(h[v]) / static_cast<double>(batches);
  });
}

// The oracle policy's retrospective access counts (sweep pass 1,
// commsim.cpp:155-166): counts[k*n + v] = number of minibatches of partition k
// over the epochs whose all_vertices contain v.
int vk_access_counts(vk_graph g, const uint8_t* roles, const uint32_t* part_of, uint32_t K, const uint32_t* fanouts,
                     uint32_t num_hops, uint64_t batch_size, uint64_t epochs, uint64_t global_seed,
                     double* counts) {
  return guard([&] {
    if (!g || !roles || !part_of || !fanouts || !counts) raise(VK_ERR_PARAMETER, "null argument");
    if (K == 0) raise(VK_ERR_PARAMETER, "need at least one partition");
    if (batch_size == 0) raise(VK_ERR_PARAMETER, "batch size must be >= 1");
    const std::uint64_t n = g->n;
    for (std::uint64_t v = 0; v < n; ++v)
      if (part_of[v] >= K) raise(VK_ERR_FORMAT, "partition label out of range");
    DeviceGuard dg(g->device);
    DevBuf hits(std::max<std::uint64_t>(1, (std::uint64_t)K * n * 4));
    VK_CUDA(cudaMemset(hits.p, 0, hits.bytes));
    VK_CUDA(cudaDeviceSynchronize());
    std::vector<std::uint32_t> parts(K);
    for (std::uint32_t k = 0; k < K; ++k) parts[k] = k;
    stream_expansions(g, roles, part_of, K, parts, fanouts, num_hops, batch_size, epochs, global_seed, nullptr, 128u,
                      [&](const std::uint32_t* all, std::uint64_t stride, const std::uint32_t* count,
                          std::uint32_t nmb, const std::uint32_t* cell_of, cudaStream_t st) {
                        // minibatches of one wave may belong to several partitions
                        std::uint32_t i = 0;
                        while (i < nmb) {
                          const std::uint32_t k = cell_of[i] % K;
                          std::uint32_t j = i;
                          while (j < nmb && cell_of[j] % K == k) ++j;
                          const unsigned gx = (unsigned)std::max<std::uint64_t>(
                              1, std::min<std::uint64_t>(ceil_div(stride, 256 * 8), 64));
                          k_histogram<<<dim3(gx, j - i), 256, 0, st>>>(all + i * stride, stride, count + i,
                                                                      hits.as<unsigned>() + (std::uint64_t)k * n);
                          count_launch();
                          VK_LAUNCH_CHECK();
                          i = j;
                        }
                      });
    std::vector<unsigned> h((std::uint64_t)K * n);
    if (!h.empty()) VK_CUDA(cudaMemcpy(h.data(), hits.p, h.size() * 4, cudaMemcpyDeviceToHost));
    for (std::size_t i = 0; i < h.size(); ++i) counts[i] = (double)h[i];
  });
}

}  // extern "C"
