// vipkit_b200 C++ mirror of the reference hot-path API.
//
// Drop-in for the reference's `namespace vipkit` declarations on this path
// (/root/reference/proj/include/vipkit/{error,rng,graph,sampling,vip,
// policies,reorder}.hpp): same type names, function names, argument meaning
// and exception types, implemented by the B200 C ABI (include/vipkit_b200.h,
// libvipkit_b200.so). Header-only; link with -lvipkit_b200.
//
//   #include <vipkit_b200/vipkit.hpp>     // instead of <vipkit/vip.hpp> ...
//   vipkit::Graph g = vipkit::load_binary_csr("g.vcsr");
//   auto scores = vipkit::propagate(g, tm, vipkit::initial_probs(roles, part, k, 1024), k);
//
// Differences (documented in INTEGRATION.md): the Graph keeps a device copy,
// created on first use (the reference Graph is immutable, graph.hpp:17-19);
// propagate_all() batches all partitions in one pass; expand_wave() and
// FeatureStore are the batched / feature-gather entry points the reference
// does not have.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <initializer_list>
#include <ostream>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../vipkit_b200.h"

namespace vipkit {

// ---- error.hpp:8-38 -------------------------------------------------------
struct error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct parse_error : error { using error::error; };
struct range_error : error { using error::error; };
struct parameter_error : error { using error::error; };
struct format_error : error { using error::error; };
struct partition_error : error { using error::error; };
struct sampling_error : error { using error::error; };
struct config_error : error { using error::error; };
struct shape_error : error { using error::error; };
struct io_error : error { using error::error; };
struct device_error : error { using error::error; };  // CUDA / unsupported (no reference twin)

namespace detail {
inline void check(int rc) {
  if (rc == VK_OK) return;
  const std::string msg = vk_last_error();
  switch (rc) {
    case VK_ERR_PARSE: throw parse_error(msg);
    case VK_ERR_RANGE: throw range_error(msg);
    case VK_ERR_PARAMETER: throw parameter_error(msg);
    case VK_ERR_FORMAT: throw format_error(msg);
    case VK_ERR_PARTITION: throw partition_error(msg);
    case VK_ERR_SAMPLING: throw sampling_error(msg);
    case VK_ERR_CONFIG: throw config_error(msg);
    case VK_ERR_SHAPE: throw shape_error(msg);
    case VK_ERR_IO: throw io_error(msg);
    default: throw device_error(std::string(vk_status_name(rc)) + ": " + msg);
  }
}
}  // namespace detail

// ---- rng.hpp:9-74 (host side; the device twin is csrc/rng.cuh) -------------
inline std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// Restated from the reference (rng.hpp:9-74): the stream definition is the
// bit-exact sampling contract, so it is the reference's, not a new design.
class RngStream {
 public:
  explicit RngStream(std::uint64_t key) : counter_(mix64(key)) {}
  std::uint64_t next_u64() {
    counter_ += 0x9e3779b97f4a7c15ull;
    std::uint64_t x = counter_;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  std::uint64_t next_below(std::uint64_t bound) {
    const std::uint64_t limit = ~0ull - ~0ull % bound;
    std::uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % bound;
  }
  /// The Weyl counter (the stream's whole state), for the device sample_neighbors.
  std::uint64_t& state() { return counter_; }

 private:
  std::uint64_t counter_;
};
namespace stream_tag {
constexpr std::uint64_t synthesis = 0xA1, roles = 0xA2, partitioning = 0xA3, minibatch_perm = 0xB1,
                        neighbor_sample = 0xB2, empirical_vip = 0xC1;
}
struct SeedSpec {
  std::uint64_t global_seed = 0;
  SeedSpec derived(std::uint64_t tag) const { return SeedSpec{mix64(global_seed ^ mix64(tag))}; }
  std::uint64_t key(std::initializer_list<std::uint64_t> parts) const {
    std::uint64_t h = global_seed;
    for (std::uint64_t p : parts) h = mix64(h ^ mix64(p));
    return h;
  }
  RngStream stream(std::initializer_list<std::uint64_t> parts) const { return RngStream(key(parts)); }
};

// ---- graph.hpp:14-69 --------------------------------------------------------
using vertex_t = std::uint32_t;
using offset_t = std::uint64_t;

struct Graph {
  std::vector<offset_t> fwd_offsets{0};
  std::vector<vertex_t> fwd_targets;
  std::vector<offset_t> rev_offsets{0};
  std::vector<vertex_t> rev_targets;
  int device = 0;  // CUDA device that holds the device copy

  std::size_t num_vertices() const { return fwd_offsets.size() - 1; }
  std::size_t num_edges() const { return fwd_targets.size(); }
  std::uint64_t out_degree(vertex_t v) const { return fwd_offsets[v + 1] - fwd_offsets[v]; }
  std::uint64_t in_degree(vertex_t v) const { return rev_offsets[v + 1] - rev_offsets[v]; }
  std::span<const vertex_t> out_neighbors(vertex_t v) const {
    return {fwd_targets.data() + fwd_offsets[v], fwd_targets.data() + fwd_offsets[v + 1]};
  }
  std::span<const vertex_t> in_neighbors(vertex_t v) const {
    return {rev_targets.data() + rev_offsets[v], rev_targets.data() + rev_offsets[v + 1]};
  }

  /// Take ownership of an existing device copy of this graph.
  void adopt(vk_graph h) { dev_ = std::shared_ptr<vk_graph_s>(h, [](vk_graph p) { vk_graph_destroy(p); }); }

  /// Device copy (created on first use; the Graph is immutable by contract).
  vk_graph handle() const {
    if (!dev_) {
      const bool have_rev = rev_offsets.size() == fwd_offsets.size() && rev_targets.size() == fwd_targets.size();
      vk_graph h = nullptr;
      detail::check(vk_graph_create(device, num_vertices(), num_edges(), fwd_offsets.data(),
                                    fwd_targets.data(), have_rev ? rev_offsets.data() : nullptr,
                                    have_rev ? rev_targets.data() : nullptr, 0, &h));
      dev_ = std::shared_ptr<vk_graph_s>(h, [](vk_graph p) { vk_graph_destroy(p); });
    }
    return dev_.get();
  }

 private:
  mutable std::shared_ptr<vk_graph_s> dev_;
};

enum class Role : std::uint8_t { train = 0, valid = 1, test = 2, none = 3 };

struct VertexRoles {
  std::vector<std::uint8_t> role;
  std::size_t size() const { return role.size(); }
  bool is_train(vertex_t v) const { return role[v] == static_cast<std::uint8_t>(Role::train); }
  std::vector<vertex_t> train_vertices() const {  // graph.cpp:77-82
    std::vector<vertex_t> out;
    for (std::size_t v = 0; v < role.size(); ++v)
      if (is_train(static_cast<vertex_t>(v))) out.push_back(static_cast<vertex_t>(v));
    return out;
  }
  std::size_t train_count() const {
    return static_cast<std::size_t>(std::count(role.begin(), role.end(), static_cast<std::uint8_t>(Role::train)));
  }
};

struct PartitionMap {
  std::uint32_t K = 1;
  std::vector<std::uint32_t> part_of;
  std::vector<std::vector<vertex_t>> members;

  // Restated from graph.cpp:88-104, error strings included: the exception
  // types and messages are part of the API callers match on.
  static PartitionMap from_labels(std::vector<std::uint32_t> labels, std::uint32_t K) {  // graph.cpp:88-104
    if (K == 0) throw parameter_error("partition count must be >= 1");
    PartitionMap pm;
    pm.K = K;
    pm.part_of = std::move(labels);
    pm.members.assign(K, {});
    for (std::size_t v = 0; v < pm.part_of.size(); ++v) {
      if (pm.part_of[v] >= K)
        throw format_error("partition label " + std::to_string(pm.part_of[v]) + " out of range for K=" +
                           std::to_string(K));
      pm.members[pm.part_of[v]].push_back(static_cast<vertex_t>(v));
    }
    for (std::uint32_t k = 0; k < K; ++k)
      if (pm.members[k].empty()) throw partition_error("partition " + std::to_string(k) + " is empty");
    return pm;
  }
  /// graph.hpp:68 (graph.cpp:106-111): partition k's train vertices, ascending.
  std::vector<vertex_t> train_members(const VertexRoles& roles, std::uint32_t k) const {
    std::vector<vertex_t> out(part_of.size());
    std::uint64_t cnt = 0;
    detail::check(vk_train_members(part_of.size(), roles.role.data(), part_of.data(), k, out.data(), &cnt));
    out.resize(cnt);
    return out;
  }
};

/// load_binary_csr (graph.hpp:117): parsed on the host, validated and the
/// reverse CSR rebuilt on the device (graph.cpp:587-596); the returned Graph
/// holds host copies (as the reference's does) and keeps the device copy.
inline Graph load_binary_csr(const std::string& path, int device = 0) {
  vk_graph h = nullptr;
  detail::check(vk_graph_load_vcsr(device, path.c_str(), 0, &h));
  std::uint64_t n = 0, m = 0;
  int sym = 0, dev = 0;
  detail::check(vk_graph_info(h, &n, &m, &sym, &dev));
  Graph g;
  g.device = device;
  g.fwd_offsets.resize(n + 1);
  g.fwd_targets.resize(m);
  g.rev_offsets.resize(n + 1);
  g.rev_targets.resize(m);
  detail::check(vk_graph_copy_forward(h, g.fwd_offsets.data(), g.fwd_targets.data()));
  detail::check(vk_graph_copy_reverse(h, g.rev_offsets.data(), g.rev_targets.data()));
  g.adopt(h);
  return g;
}

/// write_binary_csr (graph.hpp:116): the VCSR file load_binary_csr reads.
inline void write_binary_csr(const Graph& g, const std::string& path) {
  detail::check(vk_write_vcsr(path.c_str(), g.num_vertices(), g.num_edges(), g.fwd_offsets.data(),
                              g.fwd_targets.data()));
}

/// partition_from_file (graph.hpp:105): n label lines; K == 0 infers max + 1.
inline PartitionMap partition_from_file(const std::string& path, std::uint32_t K, std::size_t n) {
  std::vector<std::uint32_t> labels(n);
  std::uint32_t k_out = 0;
  detail::check(vk_partition_from_file(path.c_str(), K, n, labels.data(), &k_out));
  return PartitionMap::from_labels(std::move(labels), k_out);
}
inline void write_partition_labels(const PartitionMap& part, const std::string& path) {  // graph.hpp:122
  detail::check(vk_write_partition_labels(path.c_str(), part.part_of.data(), part.part_of.size()));
}
inline VertexRoles load_roles(const std::string& path) {  // graph.hpp:119
  std::uint8_t* r = nullptr;
  std::uint64_t n = 0;
  detail::check(vk_load_roles(path.c_str(), &r, &n));
  VertexRoles roles;
  roles.role.assign(r, r + n);
  vk_host_free(r);
  return roles;
}
inline void write_roles(const VertexRoles& roles, const std::string& path) {  // graph.hpp:120
  detail::check(vk_write_roles(path.c_str(), roles.role.data(), roles.role.size()));
}

// ---- sampling.hpp:14-64 ------------------------------------------------------
struct FanoutSpec {
  std::vector<std::uint32_t> fanouts;
  std::size_t hops() const { return fanouts.size(); }
  void validate() const {  // sampling.cpp:11-15
    if (fanouts.empty()) throw parameter_error("fanout list must have at least one hop");
    for (std::uint32_t f : fanouts)
      if (f < 1) throw parameter_error("each fanout must be >= 1");
  }
  std::string label() const {
    std::string s;
    for (std::size_t i = 0; i < fanouts.size(); ++i) s += (i ? "-" : "") + std::to_string(fanouts[i]);
    return s;
  }
};

struct ExpandedNeighborhood {
  std::vector<vertex_t> batch;
  std::vector<std::vector<vertex_t>> frontier;
  std::vector<vertex_t> all_vertices;
  // MFG (builder contract): per hop h, row pointers over the
  // sources of hop h and the index of each sampled vertex in frontier[h-1].
  std::vector<std::vector<std::uint64_t>> mfg_indptr;
  std::vector<std::vector<std::uint32_t>> mfg_dst;
};

struct BatchRef {
  std::uint64_t epoch = 0;
  std::uint32_t partition = 0;
  std::uint64_t batch_index = 0;
};

inline std::vector<std::vector<vertex_t>> epoch_minibatches(const VertexRoles& roles, const PartitionMap& part,
                                                            std::uint32_t k, std::uint64_t b, std::uint64_t epoch,
                                                            const SeedSpec& seeds,
                                                            const std::vector<vertex_t>* seed_keys = nullptr) {
  std::vector<vertex_t> perm(roles.size());
  std::uint64_t cnt = 0;
  detail::check(vk_epoch_minibatches(roles.size(), roles.role.data(), part.part_of.data(), k, b, epoch,
                                     seeds.global_seed, seed_keys ? seed_keys->data() : nullptr, perm.data(),
                                     &cnt));
  std::vector<std::vector<vertex_t>> out;
  for (std::uint64_t pos = 0; pos < cnt; pos += b)
    out.emplace_back(perm.begin() + pos, perm.begin() + std::min<std::uint64_t>(cnt, pos + b));
  return out;
}

/// Batched expand: the device sampler for a wave of minibatches.
class Sampler {
 public:
  Sampler(const Graph& g, const FanoutSpec& f, std::uint64_t batch_size, std::uint32_t max_minibatches,
          const SeedSpec& seeds) {
    f.validate();
    if (f.hops() > VK_MAX_HOPS) throw device_error("at most 8 hops are supported");
    vk_sampler_config cfg{};
    cfg.num_hops = static_cast<std::uint32_t>(f.hops());
    for (std::size_t h = 0; h < f.hops(); ++h) cfg.fanouts[h] = f.fanouts[h];
    cfg.batch_size = batch_size;
    cfg.max_minibatches = max_minibatches;
    cfg.global_seed = seeds.global_seed;
    vk_sampler s = nullptr;
    detail::check(vk_sampler_create(g.handle(), &cfg, &s));
    s_ = std::shared_ptr<vk_sampler_s>(s, [](vk_sampler p) { vk_sampler_destroy(p); });
    L_ = cfg.num_hops;
  }
  void run(const std::vector<std::span<const vertex_t>>& batches, const std::vector<BatchRef>& refs) {
    if (batches.size() != refs.size()) throw shape_error("one BatchRef per minibatch");
    std::vector<std::uint32_t> cat;
    std::vector<std::uint64_t> off{0};
    std::vector<vk_batch_ref> r(refs.size());
    for (std::size_t i = 0; i < batches.size(); ++i) {
      cat.insert(cat.end(), batches[i].begin(), batches[i].end());
      off.push_back(cat.size());
      r[i] = vk_batch_ref{refs[i].epoch, refs[i].batch_index, refs[i].partition, 0};
    }
    detail::check(vk_sampler_run(s_.get(), static_cast<std::uint32_t>(refs.size()), r.data(), cat.data(),
                                 off.data(), 0, nullptr));
    nmb_ = static_cast<std::uint32_t>(refs.size());
  }
  ExpandedNeighborhood result(std::uint32_t mb) const {
    std::vector<std::uint64_t> fs(nmb_ * L_), ec(nmb_ * L_), al(nmb_);
    detail::check(vk_sampler_sizes(s_.get(), fs.data(), ec.data(), al.data()));
    ExpandedNeighborhood nb;
    vk_sampler_view v{};
    detail::check(vk_sampler_get_view(s_.get(), &v));
    std::uint32_t nbatch = 0;
    detail::check(vk_memcpy(&nbatch, v.frontier_count[0] + mb, 4, 2 /*D2H*/));
    nb.batch.resize(nbatch);
    detail::check(vk_sampler_copy_frontier(s_.get(), mb, 0, nb.batch.data()));
    for (std::uint32_t h = 1; h <= L_; ++h) {
      nb.frontier.emplace_back(fs[mb * L_ + h - 1]);
      detail::check(vk_sampler_copy_frontier(s_.get(), mb, h, nb.frontier.back().data()));
      const std::uint64_t nsrc = h == 1 ? nbatch : fs[mb * L_ + h - 2];
      nb.mfg_indptr.emplace_back(nsrc + 1);
      nb.mfg_dst.emplace_back(ec[mb * L_ + h - 1]);
      detail::check(vk_sampler_copy_mfg(s_.get(), mb, h, nb.mfg_indptr.back().data(), nb.mfg_dst.back().data()));
    }
    nb.all_vertices.resize(al[mb]);
    detail::check(vk_sampler_copy_all(s_.get(), mb, nb.all_vertices.data()));
    return nb;
  }
  vk_sampler handle() const { return s_.get(); }
  /// seed_keys replay for the following runs (nullptr: off).
  void set_seed_keys(const std::vector<vertex_t>* seed_keys) {
    detail::check(vk_sampler_set_seed_keys(s_.get(), seed_keys ? seed_keys->data() : nullptr));
  }

 private:
  std::shared_ptr<vk_sampler_s> s_;
  std::uint32_t L_ = 0, nmb_ = 0;
};

/// vipkit::expand (sampling.hpp:62-64) for one minibatch.
inline ExpandedNeighborhood expand(const Graph& g, std::span<const vertex_t> batch, const FanoutSpec& fanouts,
                                   const SeedSpec& seeds, const BatchRef& ref,
                                   const std::vector<vertex_t>* seed_keys = nullptr) {
  if (batch.empty()) throw sampling_error("cannot expand an empty batch");  // sampling.cpp:97
  if (seed_keys && seed_keys->size() != g.num_vertices()) throw shape_error("seed_keys length does not match vertex count");
  Sampler s(g, fanouts, batch.size(), 1, seeds);
  if (seed_keys) s.set_seed_keys(seed_keys);
  s.run({batch}, {ref});
  return s.result(0);
}

/// vipkit::sample_neighbors (sampling.hpp:54-56): at most `fanout` of v's
/// out-neighbours appended to `out`, drawn on the device from `stream`
/// (advanced as the reference's is).
inline void sample_neighbors(const Graph& g, vertex_t v, std::uint32_t fanout, RngStream& stream,
                             std::vector<vertex_t>& out, const std::vector<vertex_t>* seed_keys = nullptr) {
  if (v >= g.num_vertices()) throw range_error("vertex id out of range");
  std::vector<std::uint32_t> keys;
  if (seed_keys) {  // the keys of v's neighbours, in row order (argument marshalling)
    if (seed_keys->size() != g.num_vertices()) throw shape_error("seed_keys length does not match vertex count");
    for (vertex_t u : g.out_neighbors(v)) keys.push_back((*seed_keys)[u]);
  }
  const std::size_t base = out.size();
  out.resize(base + std::min<std::uint64_t>(fanout, g.out_degree(v)));
  std::uint64_t cnt = 0;
  detail::check(vk_graph_sample_neighbors(g.handle(), v, fanout, &stream.state(), seed_keys ? keys.data() : nullptr,
                                          out.data() + base, &cnt));
  out.resize(base + cnt);
}

/// append_trace (sampling.hpp:67): epoch,partition,batch_index,vertex,hop rows.
inline void append_trace(std::ostream& out, const BatchRef& ref, const ExpandedNeighborhood& nb) {
  auto row = [&](vertex_t v, std::size_t hop) {
    out << ref.epoch << ',' << ref.partition << ',' << ref.batch_index << ',' << v << ',' << hop << '\n';
  };
  for (vertex_t v : nb.batch) row(v, 0);
  for (std::size_t h = 0; h < nb.frontier.size(); ++h)
    for (vertex_t v : nb.frontier[h]) row(v, h + 1);
}

// ---- vip.hpp:15-46 -----------------------------------------------------------
struct TransitionModel {
  enum class Kind { uniform_fanout };
  Kind kind = Kind::uniform_fanout;
  FanoutSpec fanouts;
  double weight(std::size_t hop, std::uint64_t deg) const {
    const double f = static_cast<double>(fanouts.fanouts[hop - 1]);
    const double d = static_cast<double>(deg);
    return d <= f ? 1.0 : f / d;
  }
};

struct VipScores {
  std::uint32_t partition = 0;
  std::vector<double> p0;
  std::vector<std::vector<double>> hop;
  std::vector<double> total;
};

inline std::vector<double> initial_probs(const VertexRoles& roles, const PartitionMap& part, std::uint32_t k,
                                         std::uint64_t b) {
  std::vector<double> p0(roles.size());
  detail::check(vk_initial_probs(roles.size(), roles.role.data(), part.part_of.data(), k, b, p0.data()));
  return p0;
}

/// propagate for several p0 vectors in one pass over the reverse CSR.
inline std::vector<VipScores> propagate_all(const Graph& g, const TransitionModel& tm,
                                            std::vector<std::vector<double>> p0s, std::uint32_t first_partition = 0) {
  tm.fanouts.validate();
  const std::size_t n = g.num_vertices();
  const std::size_t L = tm.fanouts.hops();
  std::vector<double> cat;
  for (auto& p : p0s) {
    if (p.size() != n) throw shape_error("p0 length does not match vertex count");
    cat.insert(cat.end(), p.begin(), p.end());
  }
  const auto C = static_cast<std::uint32_t>(p0s.size());
  std::vector<double> hop(C * L * n), total(C * n);
  detail::check(vk_vip_propagate(g.handle(), tm.fanouts.fanouts.data(), static_cast<std::uint32_t>(L), C,
                                 cat.data(), hop.data(), total.data()));
  std::vector<VipScores> out(C);
  for (std::uint32_t c = 0; c < C; ++c) {
    out[c].partition = first_partition + c;
    out[c].p0 = std::move(p0s[c]);
    for (std::size_t h = 0; h < L; ++h)
      out[c].hop.emplace_back(hop.begin() + (c * L + h) * n, hop.begin() + (c * L + h + 1) * n);
    out[c].total.assign(total.begin() + c * n, total.begin() + (c + 1) * n);
  }
  return out;
}

/// vipkit::propagate (vip.hpp:45-46).
inline VipScores propagate(const Graph& g, const TransitionModel& tm, std::vector<double> p0,
                           std::uint32_t partition = 0) {
  std::vector<std::vector<double>> v;
  v.push_back(std::move(p0));
  return std::move(propagate_all(g, tm, std::move(v), partition)[0]);
}

/// write_vip_binary / load_vip_binary (vip.hpp:58-59): n little-endian f64 totals.
inline void write_vip_binary(const VipScores& scores, const std::string& path) {
  detail::check(vk_write_vip_binary(path.c_str(), scores.total.data(), scores.total.size()));
}
inline std::vector<double> load_vip_binary(const std::string& path) {
  double* v = nullptr;
  std::uint64_t n = 0;
  detail::check(vk_load_vip_binary(path.c_str(), &v, &n));
  std::vector<double> out(v, v + n);
  vk_host_free(v);
  return out;
}

// ---- policies.hpp:16-64 -------------------------------------------------------
struct Ranking {
  std::uint32_t partition = 0;
  std::vector<vertex_t> order;
  std::vector<double> score;
  double effective_alpha = -1.0;
};

inline Ranking rank_by_scores(const PartitionMap& part, std::uint32_t k, std::span<const double> scores,
                              int device = 0) {
  Ranking r;
  r.partition = k;
  const std::size_t n = part.part_of.size();
  r.order.resize(n);
  r.score.resize(n);
  std::uint64_t cnt = 0;
  detail::check(vk_rank_by_scores(device, n, part.part_of.data(), k, scores.data(), scores.size(), r.order.data(),
                                  r.score.data(), &cnt));
  r.order.resize(cnt);
  r.score.resize(cnt);
  return r;
}

namespace detail {
template <class F>
Ranking device_ranking(const Graph& g, std::uint32_t k, F&& call) {
  Ranking r;
  r.partition = k;
  r.order.resize(g.num_vertices());
  r.score.resize(g.num_vertices());
  std::uint64_t cnt = 0;
  check(call(r.order.data(), r.score.data(), &cnt));
  r.order.resize(cnt);
  r.score.resize(cnt);
  return r;
}
}  // namespace detail

/// Baseline rankings of the Fig. 3 sweep (policies.hpp:24-45) on the device.
inline Ranking rank_degree(const Graph& g, const VertexRoles& roles, const PartitionMap& part, std::uint32_t k,
                           std::size_t L) {
  return detail::device_ranking(g, k, [&](vertex_t* o, double* s, std::uint64_t* c) {
    return vk_rank_degree(g.handle(), roles.role.data(), part.part_of.data(), part.K, k,
                          static_cast<std::uint32_t>(L), o, s, c);
  });
}
inline Ranking rank_halo_1hop(const Graph& g, const PartitionMap& part, std::uint32_t k) {
  double ea = -1.0;
  Ranking r = detail::device_ranking(g, k, [&](vertex_t* o, double* s, std::uint64_t* c) {
    return vk_rank_halo_1hop(g.handle(), part.part_of.data(), part.K, k, o, s, c, &ea);
  });
  r.effective_alpha = ea;
  return r;
}
inline Ranking rank_wpr(const Graph& g, const VertexRoles& roles, const PartitionMap& part, std::uint32_t k,
                        const TransitionModel& tm, std::uint32_t iters = 5, double damping = 0.85) {
  return detail::device_ranking(g, k, [&](vertex_t* o, double* s, std::uint64_t* c) {
    return vk_rank_wpr(g.handle(), roles.role.data(), part.part_of.data(), part.K, k, tm.fanouts.fanouts.at(0),
                       iters, damping, o, s, c);
  });
}
inline Ranking rank_numpaths(const Graph& g, const VertexRoles& roles, const PartitionMap& part, std::uint32_t k,
                             std::size_t L) {
  return detail::device_ranking(g, k, [&](vertex_t* o, double* s, std::uint64_t* c) {
    return vk_rank_numpaths(g.handle(), roles.role.data(), part.part_of.data(), part.K, k,
                            static_cast<std::uint32_t>(L), o, s, c);
  });
}

struct CachePlan {
  std::uint32_t K = 1;
  double alpha = 0.0;
  std::vector<std::vector<vertex_t>> cached;
  std::vector<std::vector<std::uint64_t>> member_bits;
  bool is_cached(std::uint32_t k, vertex_t v) const { return (member_bits[k][v >> 6] >> (v & 63)) & 1u; }
  static CachePlan empty(std::uint32_t K, std::size_t n) {
    CachePlan plan;
    plan.K = K;
    plan.cached.assign(K, {});
    plan.member_bits.assign(K, std::vector<std::uint64_t>((n + 63) / 64, 0));
    return plan;
  }
};

/// build_cache (policies.cpp:149-163): the ranking prefixes are the cache.
inline CachePlan build_cache(const std::vector<Ranking>& rankings, double alpha, std::size_t n) {
  const auto K = static_cast<std::uint32_t>(rankings.size());
  if (K == 0) throw parameter_error("need at least one ranking");
  std::uint64_t cap = 0;
  detail::check(vk_cache_capacity(alpha, n, K, &cap));
  CachePlan plan = CachePlan::empty(K, n);
  plan.alpha = alpha;
  for (std::uint32_t k = 0; k < K; ++k) {
    const auto take = std::min<std::uint64_t>(cap, rankings[k].order.size());
    plan.cached[k].assign(rankings[k].order.begin(), rankings[k].order.begin() + take);
    for (vertex_t v : plan.cached[k]) plan.member_bits[k][v >> 6] |= 1ull << (v & 63);
  }
  return plan;
}

/// empirical_vip (vip.hpp:52-55): the simulated inclusion frequency of every
/// vertex over S epochs of partition k's minibatches (device sampler).
inline std::vector<double> empirical_vip(const Graph& g, const VertexRoles& roles, const PartitionMap& part,
                                         std::uint32_t k, std::uint64_t b, const FanoutSpec& fanouts,
                                         std::uint64_t S, const SeedSpec& seeds) {
  fanouts.validate();
  std::vector<double> freq(g.num_vertices());
  detail::check(vk_empirical_vip(g.handle(), roles.role.data(), part.part_of.data(), part.K, k, b,
                                 fanouts.fanouts.data(), static_cast<std::uint32_t>(fanouts.hops()), S,
                                 seeds.global_seed, freq.data()));
  return freq;
}

// ---- commsim.hpp:14-59 -----------------------------------------
/// Per-(epoch, partition) tallies of distinct neighbourhood vertices.
struct CommReport {
  std::string policy;
  double alpha = 0.0;
  std::string fanout_label;
  std::uint64_t epochs = 0;
  std::uint32_t partitions = 0;
  struct Cell {
    std::uint64_t local_hits = 0;
    std::uint64_t cache_hits = 0;
    std::uint64_t remote_misses = 0;
  };
  std::vector<Cell> cells;  // epoch-major: cells[e * partitions + k]
  Cell& at(std::uint64_t e, std::uint32_t k) { return cells[e * partitions + k]; }
  const Cell& at(std::uint64_t e, std::uint32_t k) const { return cells[e * partitions + k]; }
  std::uint64_t total_misses() const {
    std::uint64_t t = 0;
    for (const auto& c : cells) t += c.remote_misses;
    return t;
  }
  std::uint64_t total_cache_hits() const {
    std::uint64_t t = 0;
    for (const auto& c : cells) t += c.cache_hits;
    return t;
  }
  std::uint64_t total_local_hits() const {
    std::uint64_t t = 0;
    for (const auto& c : cells) t += c.local_hits;
    return t;
  }
  double avg_epoch_misses() const {
    return epochs ? static_cast<double>(total_misses()) / static_cast<double>(epochs) : 0.0;
  }
  double improvement_vs_nocache = std::numeric_limits<double>::quiet_NaN();
};

namespace detail {
inline std::vector<CommReport> simulate_plans(const Graph& g, const VertexRoles& roles, const PartitionMap& part,
                                              const FanoutSpec& fanouts, std::uint64_t b, std::uint64_t E,
                                              const SeedSpec& seeds, const std::vector<vertex_t>& ids,
                                              const std::vector<std::uint64_t>& offsets,
                                              const std::vector<std::uint64_t>* takes,
                                              const std::vector<double>& alphas,
                                              const std::vector<vertex_t>* seed_keys) {
  fanouts.validate();
  const std::uint32_t A = static_cast<std::uint32_t>(alphas.size());
  std::vector<std::uint64_t> cells(static_cast<std::size_t>(A) * E * part.K * 3);
  check(vk_simulate(g.handle(), roles.role.data(), part.part_of.data(), part.K, fanouts.fanouts.data(),
                    static_cast<std::uint32_t>(fanouts.hops()), b, E, seeds.global_seed,
                    seed_keys ? seed_keys->data() : nullptr, ids.empty() ? nullptr : ids.data(), offsets.data(), takes ? takes->data() : nullptr, A, 0,
                    cells.data()));
  std::vector<CommReport> out(A);
  for (std::uint32_t a = 0; a < A; ++a) {
    CommReport& r = out[a];
    r.alpha = alphas[a];
    r.fanout_label = fanouts.label();
    r.epochs = E;
    r.partitions = part.K;
    r.cells.resize(E * part.K);
    for (std::size_t c = 0; c < r.cells.size(); ++c) {
      const std::uint64_t* x = cells.data() + (static_cast<std::size_t>(a) * E * part.K + c) * 3;
      r.cells[c] = {x[0], x[1], x[2]};
    }
  }
  return out;
}
}  // namespace detail

struct SimulateOptions {  // commsim.hpp:42-51
  std::ostream* trace = nullptr;        // sampling trace CSV rows
  std::ostream* batch_costs = nullptr;  // per-batch class counts CSV rows
  const std::vector<vertex_t>* seed_keys = nullptr;
  // GPU-prefix split for batch-cost rows: per-partition orderings of local
  // vertices plus the resident fraction. Empty = everything on CPU.
  const std::vector<std::vector<vertex_t>>* gpu_orderings = nullptr;
  double gamma = 0.0;
};

/// simulate (commsim.hpp:56-59) on the device: every minibatch of every
/// partition for E epochs, classified against the plan. SimulateOptions:
/// seed_keys replays relabelled streams; batch_costs rows (per-minibatch
/// class counts, the GPU-prefix split included) come from the device
/// classification (vk_simulate_batches); trace rows are the device
/// expansions' batch and frontiers, in for_each_expansion order.
inline CommReport simulate(const Graph& g, const VertexRoles& roles, const PartitionMap& part,
                           const FanoutSpec& fanouts, std::uint64_t b, std::uint64_t E, const SeedSpec& seeds,
                           const CachePlan& plan, const SimulateOptions& opts = {}) {
  if (plan.K != part.K) throw config_error("cache plan partition count differs from partition map");
  std::vector<vertex_t> ids;
  std::vector<std::uint64_t> offs{0};
  for (const auto& c : plan.cached) {
    ids.insert(ids.end(), c.begin(), c.end());
    offs.push_back(ids.size());
  }
  const std::vector<vertex_t>* sk = opts.seed_keys;
  if (sk && sk->size() != g.num_vertices()) throw shape_error("seed_keys length does not match vertex count");
  CommReport report;
  if (!opts.batch_costs) {
    report = detail::simulate_plans(g, roles, part, fanouts, b, E, seeds, ids, offs, nullptr, {plan.alpha}, sk)[0];
  } else {
    fanouts.validate();
    if (opts.gpu_orderings && opts.gpu_orderings->size() != part.K)
      throw shape_error("need one GPU ordering per partition");
    std::vector<const std::uint32_t*> gp;
    std::vector<std::uint64_t> gs;
    if (opts.gpu_orderings)
      for (const auto& o : *opts.gpu_orderings) {
        gp.push_back(o.data());
        gs.push_back(o.size());
      }
    std::uint64_t total = 0;
    for (std::uint32_t k = 0; k < part.K; ++k) total += (part.train_members(roles, k).size() + b - 1) / (b ? b : 1);
    total *= E;
    std::vector<std::uint64_t> cells(E * part.K * 3), rows(std::max<std::uint64_t>(1, total) * 7);
    std::uint64_t got = 0;
    detail::check(vk_simulate_batches(g.handle(), roles.role.data(), part.part_of.data(), part.K,
                                      fanouts.fanouts.data(), static_cast<std::uint32_t>(fanouts.hops()), b, E,
                                      seeds.global_seed, sk ? sk->data() : nullptr, ids.empty() ? nullptr : ids.data(),
                                      offs.data(), opts.gpu_orderings ? gp.data() : nullptr,
                                      opts.gpu_orderings ? gs.data() : nullptr, opts.gamma, cells.data(), rows.data(),
                                      total, &got));
    report.alpha = plan.alpha;
    report.fanout_label = fanouts.label();
    report.epochs = E;
    report.partitions = part.K;
    report.cells.resize(E * part.K);
    for (std::size_t c = 0; c < report.cells.size(); ++c)
      report.cells[c] = {cells[3 * c], cells[3 * c + 1], cells[3 * c + 2]};
    for (std::uint64_t i = 0; i < got; ++i) {
      const std::uint64_t* r = rows.data() + 7 * i;
      *opts.batch_costs << r[0] << ',' << r[1] << ',' << r[2] << ',' << r[3] << ',' << r[4] << ',' << r[5] << ','
                        << r[6] << '\n';
    }
  }
  if (opts.trace) {  // for_each_expansion (commsim.cpp:45-52) through the device sampler, one wave per cell
    for (std::uint64_t e = 0; e < E; ++e)
      for (std::uint32_t k = 0; k < part.K; ++k) {
        const auto batches = epoch_minibatches(roles, part, k, b, e, seeds, sk);
        for (std::size_t i0 = 0; i0 < batches.size(); i0 += 64) {
          const std::size_t i1 = std::min(batches.size(), i0 + 64);
          Sampler s(g, fanouts, b, static_cast<std::uint32_t>(i1 - i0), seeds);
          if (sk) s.set_seed_keys(sk);
          std::vector<std::span<const vertex_t>> bs;
          std::vector<BatchRef> refs;
          for (std::size_t i = i0; i < i1; ++i) {
            bs.emplace_back(batches[i]);
            refs.push_back(BatchRef{e, k, i});
          }
          s.run(bs, refs);
          for (std::size_t i = i0; i < i1; ++i)
            append_trace(*opts.trace, refs[i - i0], s.result(static_cast<std::uint32_t>(i - i0)));
        }
      }
  }
  return report;
}

/// The alpha axis of sweep (commsim.cpp:140-259) for one ranking policy:
/// build_cache(rankings, alpha) for every alpha, all scored from one
/// expansion pass (the plans are nested ranking prefixes).
inline std::vector<CommReport> simulate_alphas(const Graph& g, const VertexRoles& roles, const PartitionMap& part,
                                               const FanoutSpec& fanouts, std::uint64_t b, std::uint64_t E,
                                               const SeedSpec& seeds, const std::vector<Ranking>& rankings,
                                               const std::vector<double>& alphas) {
  if (rankings.size() != part.K) throw config_error("need one ranking per partition");
  if (alphas.empty() || alphas.size() > 32) throw parameter_error("between 1 and 32 alphas per pass");
  std::vector<vertex_t> ids;
  std::vector<std::uint64_t> offs{0}, takes;
  std::uint64_t cap_max = 0;
  for (double a : alphas) {
    std::uint64_t cap = 0;
    detail::check(vk_cache_capacity(a, part.part_of.size(), part.K, &cap));
    cap_max = std::max(cap_max, cap);
  }
  for (const auto& r : rankings) {
    const auto take = std::min<std::uint64_t>(cap_max, r.order.size());
    ids.insert(ids.end(), r.order.begin(), r.order.begin() + take);
    offs.push_back(ids.size());
  }
  for (double a : alphas) {
    std::uint64_t cap = 0;
    detail::check(vk_cache_capacity(a, part.part_of.size(), part.K, &cap));
    for (const auto& r : rankings) takes.push_back(std::min<std::uint64_t>(cap, r.order.size()));
  }
  return detail::simulate_plans(g, roles, part, fanouts, b, E, seeds, ids, offs, &takes, alphas, nullptr);
}

// ---- sweep (commsim.hpp:62-100, commsim.cpp:140-259) --------------------------
inline const std::vector<std::string> kAllPolicies = {"deg", "1hop", "wpr", "numpaths", "sim", "vip", "oracle"};

struct SweepConfig {
  std::vector<FanoutSpec> fanouts;
  std::uint64_t batch_size = 0;
  std::uint64_t epochs = 0;
  std::vector<double> alphas;
  std::vector<std::string> policies;
  SeedSpec seeds;
  std::uint64_t sim_epochs = 2;  // epochs behind the "sim" policy estimate
};

struct SweepResult {
  std::vector<CommReport> reports;
  struct Geomean {
    std::string policy;
    double alpha;
    double geomean_improvement;
  };
  std::vector<Geomean> geomeans;
};

// Restated from commsim.cpp:129-138 (the sweep's summary statistic).
inline double geometric_mean(std::span<const double> xs) {  // commsim.cpp:129-138
  if (xs.empty()) throw parameter_error("geometric mean of empty set");
  double log_sum = 0.0;
  for (double x : xs) {
    if (std::isinf(x)) return x;
    if (!(x > 0)) throw parameter_error("geometric mean needs positive values");
    log_sum += std::log(x);
  }
  return std::exp(log_sum / static_cast<double>(xs.size()));
}

/// The policy x alpha x fanout grid on the device: every ranking, the
/// oracle's access counts and each policy's alpha axis (vk_simulate) run on
/// the GPU; expansions are identical across plans by construction. The
/// control flow (grid loops, no-cache baseline, improvement and geomean
/// bookkeeping) follows commsim.cpp:140-259 so the SweepResult matches the
/// reference's; the per-cell work is replaced by the device calls.
inline SweepResult sweep(const Graph& g, const VertexRoles& roles, const PartitionMap& part,
                         const SweepConfig& cfg) {
  if (cfg.fanouts.empty() || cfg.alphas.empty() || cfg.policies.empty())
    throw parameter_error("sweep needs non-empty fanout, alpha, and policy grids");
  for (const auto& p : cfg.policies)
    if (std::find(kAllPolicies.begin(), kAllPolicies.end(), p) == kAllPolicies.end())
      throw parameter_error("unknown policy: " + p);
  const std::size_t n = g.num_vertices();
  SweepResult result;
  std::vector<std::vector<std::vector<double>>> improvements(
      cfg.policies.size(), std::vector<std::vector<double>>(cfg.alphas.size()));
  for (const FanoutSpec& fanouts : cfg.fanouts) {
    fanouts.validate();
    const std::size_t L = fanouts.hops();
    const TransitionModel tm{TransitionModel::Kind::uniform_fanout, fanouts};
    std::vector<double> access;
    if (std::find(cfg.policies.begin(), cfg.policies.end(), "oracle") != cfg.policies.end()) {
      access.resize(part.K * n);
      detail::check(vk_access_counts(g.handle(), roles.role.data(), part.part_of.data(), part.K,
                                     fanouts.fanouts.data(), static_cast<std::uint32_t>(L), cfg.batch_size,
                                     cfg.epochs, cfg.seeds.global_seed, access.data()));
    }
    std::vector<CommReport> reports;
    for (const std::string& policy : cfg.policies) {
      std::vector<Ranking> rk;
      for (std::uint32_t k = 0; k < part.K; ++k) {
        if (policy == "deg")
          rk.push_back(rank_degree(g, roles, part, k, L));
        else if (policy == "1hop")
          rk.push_back(rank_halo_1hop(g, part, k));
        else if (policy == "wpr")
          rk.push_back(rank_wpr(g, roles, part, k, tm));
        else if (policy == "numpaths")
          rk.push_back(rank_numpaths(g, roles, part, k, L));
        else if (policy == "sim")
          rk.push_back(rank_by_scores(
              part, k, empirical_vip(g, roles, part, k, cfg.batch_size, fanouts, cfg.sim_epochs, cfg.seeds),
              g.device));
        else if (policy == "vip")
          rk.push_back(rank_by_scores(
              part, k, propagate(g, tm, initial_probs(roles, part, k, cfg.batch_size), k).total, g.device));
        else  // oracle
          rk.push_back(rank_by_scores(part, k, std::span<const double>(access.data() + k * n, n), g.device));
      }
      auto r = simulate_alphas(g, roles, part, fanouts, cfg.batch_size, cfg.epochs, cfg.seeds, rk, cfg.alphas);
      for (auto& x : r) x.policy = policy;
      reports.insert(reports.end(), r.begin(), r.end());
    }
    // no-cache baseline: every cache hit of any report is a miss without it
    const std::uint64_t base = reports[0].total_cache_hits() + reports[0].total_misses();
    for (std::size_t p = 0; p < cfg.policies.size(); ++p)
      for (std::size_t a = 0; a < cfg.alphas.size(); ++a) {
        CommReport& r = reports[p * cfg.alphas.size() + a];
        const auto misses = r.total_misses();
        if (base == 0)
          r.improvement_vs_nocache = 1.0;
        else if (misses == 0)
          r.improvement_vs_nocache = std::numeric_limits<double>::infinity();
        else
          r.improvement_vs_nocache = static_cast<double>(base) / static_cast<double>(misses);
        improvements[p][a].push_back(r.improvement_vs_nocache);
        result.reports.push_back(std::move(r));
      }
  }
  for (std::size_t p = 0; p < cfg.policies.size(); ++p)
    for (std::size_t a = 0; a < cfg.alphas.size(); ++a)
      result.geomeans.push_back({cfg.policies[p], cfg.alphas[a], geometric_mean(improvements[p][a])});
  return result;
}

// ---- reorder.hpp:15-26 --------------------------------------------------------
struct ReorderMap {
  std::vector<vertex_t> new_of_old;
  std::vector<vertex_t> old_of_new;
  std::vector<std::pair<std::uint64_t, std::uint64_t>> ranges;
  std::size_t size() const { return new_of_old.size(); }
};

inline ReorderMap build_reorder(const PartitionMap& part, const std::vector<std::vector<double>>& scores,
                                int device = 0) {
  if (scores.size() != part.K) throw shape_error("need one score vector per partition");
  const std::size_t n = part.part_of.size();
  std::vector<double> cat;
  for (const auto& s : scores) {
    if (s.size() != n) throw shape_error("score vector length does not match vertex count");
    cat.insert(cat.end(), s.begin(), s.end());
  }
  ReorderMap m;
  m.old_of_new.resize(n);
  std::vector<std::uint64_t> ranges(2 * part.K);
  detail::check(vk_build_reorder(device, n, part.K, part.part_of.data(), cat.data(), m.old_of_new.data(),
                                 ranges.data()));
  m.new_of_old.resize(n);
  for (std::size_t i = 0; i < n; ++i) m.new_of_old[m.old_of_new[i]] = static_cast<vertex_t>(i);
  for (std::uint32_t k = 0; k < part.K; ++k) m.ranges.emplace_back(ranges[2 * k], ranges[2 * k + 1]);
  return m;
}

struct ReorderedDataset {
  Graph graph;
  VertexRoles roles;
  PartitionMap part;
};

/// apply_reorder (reorder.hpp:34-35): the relabelled graph is built on the
/// device (vk_graph_apply_reorder); roles and labels permute on the host.
inline ReorderedDataset apply_reorder(const Graph& g, const VertexRoles& roles, const PartitionMap& part,
                                      const ReorderMap& map) {
  const std::size_t n = g.num_vertices();
  if (map.size() != n) throw shape_error("reorder map size does not match vertex count");  // reorder.cpp:39
  vk_graph h = nullptr;
  detail::check(vk_graph_apply_reorder(g.handle(), map.old_of_new.data(), &h));
  ReorderedDataset out;
  Graph& ng = out.graph;
  ng.device = g.device;
  std::uint64_t nn = 0, m = 0;
  int sym = 0, dev = 0;
  detail::check(vk_graph_info(h, &nn, &m, &sym, &dev));
  ng.fwd_offsets.resize(n + 1);
  ng.fwd_targets.resize(m);
  ng.rev_offsets.resize(n + 1);
  ng.rev_targets.resize(m);
  detail::check(vk_graph_copy_forward(h, ng.fwd_offsets.data(), ng.fwd_targets.data()));
  detail::check(vk_graph_copy_reverse(h, ng.rev_offsets.data(), ng.rev_targets.data()));
  ng.adopt(h);
  out.roles.role.resize(n);
  std::vector<std::uint32_t> labels(n);
  for (std::size_t u = 0; u < n; ++u) {
    out.roles.role[u] = roles.role[map.old_of_new[u]];
    labels[u] = part.part_of[map.old_of_new[u]];
  }
  out.part = PartitionMap::from_labels(std::move(labels), part.K);
  return out;
}

// ---- feature gather (new: the reference never materialises features) -------
class FeatureStore {
 public:
  FeatureStore(const PartitionMap& part, const ReorderMap& map, std::uint32_t dim, int dtype = VK_F32,
               int device = 0) {
    std::vector<std::uint64_t> r;
    for (auto& [a, b] : map.ranges) {
      r.push_back(a);
      r.push_back(b);
    }
    vk_plane p = nullptr;
    detail::check(vk_plane_create(device, part.part_of.size(), part.K, dim, dtype, part.part_of.data(),
                                  map.old_of_new.data(), r.data(), &p));
    p_ = std::shared_ptr<vk_plane_s>(p, [](vk_plane q) { vk_plane_destroy(q); });
  }
  void load_partition(std::uint32_t k, const std::vector<vertex_t>& cached, const void* features,
                      std::uint64_t feature_seed = 0) {
    detail::check(vk_plane_load_partition(p_.get(), k, cached.data(), cached.size(), features, feature_seed));
  }
  bool is_cached(std::uint32_t k, vertex_t v) const {
    int out = 0;
    detail::check(vk_plane_is_cached(p_.get(), k, v, &out));
    return out != 0;
  }
  /// classify + gather for the sampler's last wave into device memory.
  void gather(const Sampler& s, void* out_dev, std::uint64_t out_stride_rows, std::uint64_t* counts_dev,
              vk_stream_t stream = nullptr) {
    detail::check(vk_plane_gather(p_.get(), s.handle(), out_dev, out_stride_rows, counts_dev, stream));
  }
  vk_plane handle() const { return p_.get(); }

 private:
  std::shared_ptr<vk_plane_s> p_;
};

}  // namespace vipkit
