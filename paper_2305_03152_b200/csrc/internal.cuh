// Internal handle layouts shared by the library's translation units.
#pragma once
#include <atomic>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace vk {
extern std::atomic<std::uint64_t> g_launches;
inline void count_launch(std::uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
// epoch_minibatches' shuffle of partition k's train members (capi.cu)
void epoch_shuffle(std::uint32_t* perm, std::uint64_t T, std::uint32_t k, std::uint64_t epoch,
                   std::uint64_t global_seed);
}  // namespace vk

// Device-resident graph (replaces vipkit::Graph, graph.hpp:20-46). Offsets
// u64 [n+1], targets u32 [m]; for undirected graphs the reverse structure
// aliases the forward one, halving HBM footprint.
struct vk_graph_s {
  int device = 0;
  std::uint64_t n = 0, m = 0;
  bool symmetric = false;
  std::uint32_t max_out_degree = 0;
  vk::DevBuf fwd_off, fwd_tgt;
  vk::DevBuf rev_off_buf, rev_tgt_buf;
  const std::uint64_t* rev_off = nullptr;
  const std::uint32_t* rev_tgt = nullptr;
  vk::DevBuf out_deg;  // u32 [n] forward (out) degrees: TransitionModel::weight input

  // VIP pull schedule: rows grouped by in-degree class, each class listed in
  // ascending row order (vip.cu).
  bool sched_ready = false;
  vk::DevBuf sched_rows;                     // u32 [n]
  std::vector<std::uint64_t> sched_offsets;  // class boundaries in sched_rows
  cudaStream_t stream = nullptr;
  // VIP workspace, grown on demand and kept across calls (no allocation on
  // the timed path).
  vk::DevBuf vip_lm_a, vip_lm_b, vip_partial, vip_flag, vip_active;
  bool vip_last_f32 = false;  // storage width used by the last propagate (diagnostics)

  const std::uint64_t* d_off() const { return fwd_off.as<std::uint64_t>(); }
  const std::uint32_t* d_tgt() const { return fwd_tgt.as<std::uint32_t>(); }
};

namespace vk {
void build_vip_schedule(vk_graph_s& g);
}
