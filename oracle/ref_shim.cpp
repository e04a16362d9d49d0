// TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/src. It exists so the Python test-suite and bench.py's
// CPU-baseline leg can call the real reference (vipkit::*) with plain arrays.
// Every entry point forwards to the reference function named in its comment.
// Three pieces are not single calls, and say so where they are defined:
// ref_expand's MFG edge list drives the reference's own `SeedSpec::stream` +
// `sample_neighbors` exactly as `expand` does (sampling.cpp:106-114), because
// the reference has no MFG output; the CPU-arm drivers restate `classify`
// (commsim.cpp:61-73, in an anonymous namespace there, so not callable) and
// the row gather out[i] = X[all[i]] (not in the reference at all).
#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "vipkit/commsim.hpp"
#include "vipkit/error.hpp"
#include "vipkit/graph.hpp"
#include "vipkit/parallel.hpp"
#include "vipkit/policies.hpp"
#include "vipkit/reorder.hpp"
#include "vipkit/rng.hpp"
#include "vipkit/sampling.hpp"
#include "vipkit/vip.hpp"

using namespace vipkit;

namespace {

thread_local std::string g_err;

// libstdc++ is linked statically into this .so: construct the standard
// streams' locale state at load time so the reference's formatted ofstream
// writers (write_roles, simulate's CSV streams) work when dlopen'ed.
const std::ios_base::Init g_ios_init;

// Same numbering as include/vipkit_b200.h (vk_status).
int code_of(const std::exception& e) {
  if (dynamic_cast<const parse_error*>(&e)) return 1;
  if (dynamic_cast<const range_error*>(&e)) return 2;
  if (dynamic_cast<const parameter_error*>(&e)) return 3;
  if (dynamic_cast<const format_error*>(&e)) return 4;
  if (dynamic_cast<const partition_error*>(&e)) return 5;
  if (dynamic_cast<const sampling_error*>(&e)) return 6;
  if (dynamic_cast<const config_error*>(&e)) return 7;
  if (dynamic_cast<const shape_error*>(&e)) return 8;
  if (dynamic_cast<const io_error*>(&e)) return 9;
  return 23;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

VertexRoles make_roles_view(const std::uint8_t* roles, std::uint64_t n) {
  VertexRoles r;
  r.role.assign(roles, roles + n);
  return r;
}

PartitionMap make_part(const std::uint32_t* labels, std::uint64_t n, std::uint32_t K) {
  return PartitionMap::from_labels(std::vector<std::uint32_t>(labels, labels + n), K);
}

FanoutSpec make_fanouts(const std::uint32_t* f, std::uint32_t L) {
  FanoutSpec s;
  s.fanouts.assign(f, f + L);
  return s;
}

// Static-chunked worker pool for the CPU-baseline driver (the reference's
// own parallel_for splits one index range the same way, parallel.hpp:17-39).
template <class F>
void parallel_for_workers(unsigned workers, std::size_t total, F&& fn) {
  if (workers <= 1 || total < 2) {
    for (std::size_t i = 0; i < total; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  std::atomic<std::size_t> next{0};
  for (unsigned w = 0; w < workers; ++w)
    th.emplace_back([&] {
      for (std::size_t i = next++; i < total; i = next++) fn(i);
    });
  for (auto& t : th) t.join();
}

struct Expansion {
  ExpandedNeighborhood nb;
  std::vector<std::vector<std::uint64_t>> indptr;  // per hop, |F_{h-1}|+1
  std::vector<std::vector<vertex_t>> edges;        // per hop, sampled ids in draw order
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(unsigned n) { set_thread_count(n); }

// ---- graph ----
void* ref_graph_generate(int kind, std::uint64_t n, std::uint64_t d, std::uint64_t seed) {
  Graph* out = nullptr;
  const int rc = guard([&] {
    out = new Graph(generate_synthetic(static_cast<SynthKind>(kind), SynthParams{n, d, seed}));
  });
  return rc == 0 ? out : nullptr;
}

void* ref_graph_from_edges(std::uint64_t n, const std::uint32_t* src, const std::uint32_t* dst,
                           std::uint64_t ne, int undirected) {
  Graph* out = nullptr;
  const int rc = guard([&] {
    std::vector<std::pair<vertex_t, vertex_t>> e(ne);
    for (std::uint64_t i = 0; i < ne; ++i) e[i] = {src[i], dst[i]};
    out = new Graph(Graph::from_edges(n, std::move(e), undirected != 0));
  });
  return rc == 0 ? out : nullptr;
}

// Forward CSR given; the reverse CSR is rebuilt with the same transpose
// load_binary_csr performs (graph.cpp:587-596) and validated by the
// reference's own check_invariants. (Going through a VCSR temp file would be
// identical but needs a byte-wise u64 decode of m targets.)
void* ref_graph_from_csr(std::uint64_t n, std::uint64_t m, const std::uint64_t* off,
                         const std::uint32_t* tgt) {
  Graph* out = nullptr;
  const int rc = guard([&] {
    auto* g = new Graph();
    g->fwd_offsets.assign(off, off + n + 1);
    g->fwd_targets.assign(tgt, tgt + m);
    g->rev_offsets.assign(n + 1, 0);
    for (std::uint64_t i = 0; i < m; ++i) g->rev_offsets[tgt[i] + 1]++;
    for (std::uint64_t i = 0; i < n; ++i) g->rev_offsets[i + 1] += g->rev_offsets[i];
    g->rev_targets.resize(m);
    std::vector<offset_t> cursor(g->rev_offsets.begin(), g->rev_offsets.end() - 1);
    for (std::uint64_t u = 0; u < n; ++u)
      for (offset_t i = off[u]; i < off[u + 1]; ++i)
        g->rev_targets[cursor[tgt[i]]++] = static_cast<vertex_t>(u);
    g->check_invariants();  // graph.cpp:55-75
    out = g;
  });
  return rc == 0 ? out : nullptr;
}

// Undirected bench graphs (canonical symmetric CSR, sorted rows): the
// transpose load_binary_csr builds (graph.cpp:587-595) is the forward CSR
// itself, so the reverse side is a (threaded) copy instead of an O(m)
// random scatter (150 s single-threaded at papers scale). check != 0 runs the
// reference's check_invariants (graph.cpp:55-75) as well.
void* ref_graph_from_symmetric_csr(std::uint64_t n, std::uint64_t m, const std::uint64_t* off,
                                   const std::uint32_t* tgt, unsigned threads, int check) {
  Graph* out = nullptr;
  const int rc = guard([&] {
    auto* g = new Graph();
    g->fwd_offsets.assign(off, off + n + 1);
    g->rev_offsets.assign(off, off + n + 1);
    g->fwd_targets.resize(m);
    g->rev_targets.resize(m);
    const unsigned T = std::max(1u, threads);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const std::uint64_t lo = m * t / T, hi = m * (t + 1) / T;
        std::memcpy(g->fwd_targets.data() + lo, tgt + lo, (hi - lo) * 4);
        std::memcpy(g->rev_targets.data() + lo, tgt + lo, (hi - lo) * 4);
      });
    for (auto& x : th) x.join();
    if (check) g->check_invariants();
    out = g;
  });
  return rc == 0 ? out : nullptr;
}

void* ref_graph_load_vcsr(const char* path) {
  Graph* out = nullptr;
  const int rc = guard([&] { out = new Graph(load_binary_csr(path)); });  // graph.cpp:565
  return rc == 0 ? out : nullptr;
}

int ref_graph_write_vcsr(void* g, const char* path) {
  return guard([&] { write_binary_csr(*static_cast<Graph*>(g), path); });  // graph.cpp:553
}

std::uint64_t ref_graph_n(void* g) { return static_cast<Graph*>(g)->num_vertices(); }
std::uint64_t ref_graph_m(void* g) { return static_cast<Graph*>(g)->num_edges(); }

void ref_graph_copy(void* gp, std::uint64_t* off, std::uint32_t* tgt, std::uint64_t* roff,
                    std::uint32_t* rtgt) {
  const Graph& g = *static_cast<Graph*>(gp);
  if (off) std::memcpy(off, g.fwd_offsets.data(), g.fwd_offsets.size() * 8);
  if (tgt) std::memcpy(tgt, g.fwd_targets.data(), g.fwd_targets.size() * 4);
  if (roff) std::memcpy(roff, g.rev_offsets.data(), g.rev_offsets.size() * 8);
  if (rtgt) std::memcpy(rtgt, g.rev_targets.data(), g.rev_targets.size() * 4);
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

// ---- roles / partitions ----
int ref_make_roles(std::uint64_t n, double train, double valid, double test, std::uint64_t seed,
                   std::uint8_t* out) {
  return guard([&] {
    const auto r = make_roles(n, train, valid, test, seed);  // graph.cpp:247
    std::memcpy(out, r.role.data(), n);
  });
}

int ref_partition_graph(void* g, const std::uint8_t* roles, std::uint64_t n, std::uint32_t K,
                        int method, std::uint64_t seed, std::uint32_t* labels_out) {
  return guard([&] {
    const auto part = partition_graph(*static_cast<Graph*>(g), make_roles_view(roles, n), K,
                                      static_cast<PartitionMethod>(method), seed);  // graph.cpp:448
    std::memcpy(labels_out, part.part_of.data(), n * 4);
  });
}

// ---- sampling ----
// A VertexRoles + PartitionMap pair built once (as the reference's callers
// do, commsim.cpp:45-52), so per-epoch schedules cost what
// epoch_minibatches costs and not a PartitionMap rebuild.
struct RefCtx {
  VertexRoles roles;
  PartitionMap part;
};
void* ref_ctx_create(const std::uint8_t* roles, const std::uint32_t* labels, std::uint64_t n, std::uint32_t K) {
  RefCtx* out = nullptr;
  const int rc = guard([&] { out = new RefCtx{make_roles_view(roles, n), make_part(labels, n, K)}; });
  return rc == 0 ? out : nullptr;
}
void ref_ctx_free(void* c) { delete static_cast<RefCtx*>(c); }
int ref_ctx_epoch(void* c, std::uint32_t k, std::uint64_t b, std::uint64_t epoch, std::uint64_t seed,
                  std::uint32_t* out_perm, std::uint64_t* out_count) {
  return guard([&] {
    const RefCtx& x = *static_cast<RefCtx*>(c);
    const auto batches = epoch_minibatches(x.roles, x.part, k, b, epoch, SeedSpec{seed});  // sampling.cpp:45
    std::uint64_t pos = 0;
    for (const auto& bt : batches) {
      std::memcpy(out_perm + pos, bt.data(), bt.size() * 4);
      pos += bt.size();
    }
    *out_count = pos;
  });
}

// epoch_minibatches (sampling.cpp:45-70); batches are the consecutive
// b-chunks of the returned permutation.
int ref_epoch_minibatches(const std::uint8_t* roles, std::uint64_t n, const std::uint32_t* labels,
                          std::uint32_t K, std::uint32_t k, std::uint64_t b, std::uint64_t epoch,
                          std::uint64_t seed, const std::uint32_t* seed_keys,
                          std::uint32_t* out_perm, std::uint64_t* out_count) {
  return guard([&] {
    std::vector<vertex_t> keys;
    if (seed_keys) keys.assign(seed_keys, seed_keys + n);
    const auto batches =
        epoch_minibatches(make_roles_view(roles, n), make_part(labels, n, K), k, b, epoch,
                          SeedSpec{seed}, seed_keys ? &keys : nullptr);
    std::uint64_t pos = 0;
    for (const auto& bt : batches) {
      std::memcpy(out_perm + pos, bt.data(), bt.size() * 4);
      pos += bt.size();
    }
    *out_count = pos;
  });
}

void* ref_expand(void* gp, const std::uint32_t* batch, std::uint64_t nb, const std::uint32_t* fan,
                 std::uint32_t L, std::uint64_t seed, std::uint64_t epoch, std::uint32_t part,
                 std::uint64_t batch_index, int with_mfg, const std::uint32_t* seed_keys) {
  Expansion* out = nullptr;
  const int rc = guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const FanoutSpec fanouts = make_fanouts(fan, L);
    const SeedSpec seeds{seed};
    const BatchRef ref{epoch, part, batch_index};
    std::vector<vertex_t> keys;
    if (seed_keys) keys.assign(seed_keys, seed_keys + g.num_vertices());
    const std::vector<vertex_t>* sk = seed_keys ? &keys : nullptr;
    auto* x = new Expansion();
    x->nb = expand(g, std::span<const vertex_t>(batch, nb), fanouts, seeds, ref, sk);  // sampling.cpp:94
    if (with_mfg) {
      // MFG: the per-source draw sequence of expand's hop loop
      // (sampling.cpp:106-114), replayed with the reference's own stream
      // and sample_neighbors; sources in the order expand visits them.
      const std::vector<vertex_t>* cur = &x->nb.batch;
      for (std::size_t h = 1; h <= L; ++h) {
        std::vector<std::uint64_t> ip{0};
        std::vector<vertex_t> ed;
        for (vertex_t v : *cur) {
          RngStream s = seeds.stream({stream_tag::neighbor_sample, ref.epoch, ref.partition,
                                      ref.batch_index, static_cast<std::uint64_t>(h),
                                      sk ? static_cast<std::uint64_t>((*sk)[v]) : v});
          sample_neighbors(g, v, fanouts.fanouts[h - 1], s, ed, sk);
          ip.push_back(ed.size());
        }
        x->indptr.push_back(std::move(ip));
        x->edges.push_back(std::move(ed));
        cur = &x->nb.frontier[h - 1];
      }
    }
    out = x;
  });
  return rc == 0 ? out : nullptr;
}

std::uint64_t ref_exp_frontier_size(void* x, std::uint32_t h) {
  return static_cast<Expansion*>(x)->nb.frontier[h].size();
}
const std::uint32_t* ref_exp_frontier(void* x, std::uint32_t h) {
  return static_cast<Expansion*>(x)->nb.frontier[h].data();
}
std::uint64_t ref_exp_all_size(void* x) { return static_cast<Expansion*>(x)->nb.all_vertices.size(); }
const std::uint32_t* ref_exp_all(void* x) { return static_cast<Expansion*>(x)->nb.all_vertices.data(); }
std::uint64_t ref_exp_edges_size(void* x, std::uint32_t h) {
  return static_cast<Expansion*>(x)->edges[h].size();
}
const std::uint32_t* ref_exp_edges(void* x, std::uint32_t h) {
  return static_cast<Expansion*>(x)->edges[h].data();
}
const std::uint64_t* ref_exp_indptr(void* x, std::uint32_t h) {
  return static_cast<Expansion*>(x)->indptr[h].data();
}
void ref_exp_free(void* x) { delete static_cast<Expansion*>(x); }

// sample_neighbors (sampling.cpp:72-92) on a stream keyed by `key`.
int ref_sample_neighbors(void* gp, std::uint32_t v, std::uint32_t fanout, std::uint64_t key,
                         std::uint32_t* out, std::uint64_t* out_count) {
  return guard([&] {
    RngStream s(key);
    std::vector<vertex_t> o;
    sample_neighbors(*static_cast<Graph*>(gp), v, fanout, s, o);
    std::memcpy(out, o.data(), o.size() * 4);
    *out_count = o.size();
  });
}

// sample_neighbors with the stream's final state and optional seed_keys.
int ref_sample_neighbors_state(void* gp, std::uint32_t v, std::uint32_t fanout, std::uint64_t key,
                               const std::uint32_t* seed_keys, std::uint32_t* out, std::uint64_t* out_count,
                               std::uint64_t* next_draw) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    RngStream s(key);
    std::vector<vertex_t> o, keys;
    if (seed_keys) keys.assign(seed_keys, seed_keys + g.num_vertices());
    sample_neighbors(g, v, fanout, s, o, seed_keys ? &keys : nullptr);  // sampling.cpp:72-92
    std::memcpy(out, o.data(), o.size() * 4);
    *out_count = o.size();
    *next_draw = s.next_u64();  // where the stream stands afterwards
  });
}

// ---- file formats: the reference's own readers and writers ----
int ref_write_partition_labels(const std::uint32_t* labels, std::uint64_t n, std::uint32_t K, const char* path) {
  return guard([&] { write_partition_labels(make_part(labels, n, K), path); });  // graph.cpp:624
}
int ref_partition_from_file(const char* path, std::uint32_t K, std::uint64_t n, std::uint32_t* labels_out,
                            std::uint32_t* K_out) {
  return guard([&] {
    const PartitionMap pm = partition_from_file(path, K, n);  // graph.cpp:461
    std::memcpy(labels_out, pm.part_of.data(), n * 4);
    *K_out = pm.K;
  });
}
int ref_write_roles(const std::uint8_t* roles, std::uint64_t n, const char* path) {
  return guard([&] { write_roles(make_roles_view(roles, n), path); });  // graph.cpp:618
}
int ref_load_roles(const char* path, std::uint8_t* out, std::uint64_t cap, std::uint64_t* n) {
  return guard([&] {
    const VertexRoles r = load_roles(path);  // graph.cpp:600
    *n = r.role.size();
    std::memcpy(out, r.role.data(), std::min<std::uint64_t>(cap, r.role.size()));
  });
}
int ref_write_vip_binary(const double* total, std::uint64_t n, const char* path) {
  return guard([&] {
    VipScores s;
    s.total.assign(total, total + n);
    write_vip_binary(s, path);  // vip.cpp:107
  });
}
int ref_load_vip_binary(const char* path, double* out, std::uint64_t cap, std::uint64_t* n) {
  return guard([&] {
    const auto v = load_vip_binary(path);  // vip.cpp:122
    *n = v.size();
    std::memcpy(out, v.data(), std::min<std::uint64_t>(cap, v.size()) * 8);
  });
}

// Batched driver for the CPU baseline: expands minibatches [i0, i1) of one
// (epoch, partition) cell with `threads` workers over independent minibatches
// (expand is pure, sampling.cpp:82 thread_local scratch) and classifies each
// as commsim.cpp:61-73 does. Returns the summed |all_vertices| and the
// local/cache/miss tallies.
int ref_expand_classify_range(void* gp, const std::uint32_t* perm, std::uint64_t perm_count,
                              std::uint64_t b, const std::uint32_t* fan, std::uint32_t L,
                              std::uint64_t seed, std::uint64_t epoch, std::uint32_t k,
                              std::uint64_t i0, std::uint64_t i1, const std::uint32_t* labels,
                              const std::uint64_t* cache_bits /* (n+63)/64 words for k, or null */,
                              unsigned threads, std::uint64_t* tallies /* all,local,cache,miss */) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const FanoutSpec fanouts = make_fanouts(fan, L);
    const SeedSpec seeds{seed};
    const std::uint64_t nbatch = i1 - i0;
    std::vector<std::uint64_t> t(4 * nbatch, 0);
    parallel_for_workers(threads, nbatch, [&](std::size_t j) {
      const std::uint64_t i = i0 + j;
      const std::uint64_t lo = i * b;
      const std::uint64_t hi = std::min<std::uint64_t>(perm_count, lo + b);
      const auto nb = expand(g, std::span<const vertex_t>(perm + lo, hi - lo), fanouts, seeds,
                             BatchRef{epoch, k, i});
      std::uint64_t loc = 0, hit = 0, miss = 0;
      for (vertex_t v : nb.all_vertices) {
        if (labels[v] == k)
          ++loc;
        else if (cache_bits && ((cache_bits[v >> 6] >> (v & 63)) & 1u))
          ++hit;
        else
          ++miss;
      }
      t[4 * j] = nb.all_vertices.size();
      t[4 * j + 1] = loc;
      t[4 * j + 2] = hit;
      t[4 * j + 3] = miss;
    });
    for (std::uint64_t j = 0; j < nbatch; ++j)
      for (int c = 0; c < 4; ++c) tallies[c] += t[4 * j + c];
  });
}

// bench.py's CPU arms, one call per step: minibatch j (its own BatchRef
// refs[3j..3j+2] = epoch, partition, batch index, and its seeds) is expanded
// by the reference (sampling.cpp:94-128) and classified as commsim.cpp:61-73
// does (restated); with a feature table, its all_vertices rows are then
// gathered (out[i] = X[all[i]], restated: the reference has no gather) into
// the worker's slice of `work` (threads x cap rows). Workers take minibatches
// dynamically. tallies: nmb x {all, local, cache, miss}.
int ref_bench_minibatches(void* gp, std::uint32_t nmb, const std::uint32_t* seeds,
                          const std::uint64_t* seed_off, const std::uint64_t* refs, const std::uint32_t* fan,
                          std::uint32_t L, std::uint64_t seed, const std::uint32_t* labels,
                          const std::uint64_t* cache_bits /* K x W, or null */, std::uint64_t W,
                          const unsigned char* table, std::uint64_t row_bytes, unsigned char* work,
                          std::uint64_t cap, unsigned threads, std::uint64_t* tallies) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const FanoutSpec fanouts = make_fanouts(fan, L);
    const SeedSpec seeds_spec{seed};
    std::atomic<std::uint32_t> next{0};
    std::string err;
    std::atomic<bool> failed{false};
    auto worker = [&](unsigned w) {
      try {
        for (std::uint32_t j = next++; j < nmb; j = next++) {
          const std::uint32_t k = (std::uint32_t)refs[3 * j + 1];
          const auto nb = expand(g, std::span<const vertex_t>(seeds + seed_off[j], seed_off[j + 1] - seed_off[j]),
                                 fanouts, seeds_spec, BatchRef{refs[3 * j], k, refs[3 * j + 2]});
          std::uint64_t loc = 0, hit = 0, miss = 0;
          const std::uint64_t* bits = cache_bits ? cache_bits + (std::uint64_t)k * W : nullptr;
          for (vertex_t v : nb.all_vertices) {
            if (labels[v] == k)
              ++loc;
            else if (bits && ((bits[v >> 6] >> (v & 63)) & 1u))
              ++hit;
            else
              ++miss;
          }
          if (table) {
            if (nb.all_vertices.size() > cap) throw shape_error("gather buffer too small");
            unsigned char* out = work + (std::uint64_t)w * cap * row_bytes;
            for (std::size_t i = 0; i < nb.all_vertices.size(); ++i)
              std::memcpy(out + i * row_bytes, table + (std::uint64_t)nb.all_vertices[i] * row_bytes, row_bytes);
          }
          tallies[4 * j] = nb.all_vertices.size();
          tallies[4 * j + 1] = loc;
          tallies[4 * j + 2] = hit;
          tallies[4 * j + 3] = miss;
        }
      } catch (const std::exception& e) {
        if (!failed.exchange(true)) err = e.what();
      }
    };
    const unsigned T = std::max(1u, std::min<unsigned>(threads, nmb));
    std::vector<std::thread> th;
    for (unsigned w = 1; w < T; ++w) th.emplace_back(worker, w);
    worker(0);
    for (auto& t : th) t.join();
    if (failed) throw parameter_error(err);
  });
}

// ---- vip ----
int ref_initial_probs(const std::uint8_t* roles, std::uint64_t n, const std::uint32_t* labels,
                      std::uint32_t K, std::uint32_t k, std::uint64_t b, double* out) {
  return guard([&] {
    const auto p0 = initial_probs(make_roles_view(roles, n), make_part(labels, n, K), k, b);  // vip.cpp:25
    std::memcpy(out, p0.data(), n * 8);
  });
}

int ref_propagate(void* gp, const std::uint32_t* fan, std::uint32_t L, const double* p0,
                  double* hop_out, double* total_out) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const std::uint64_t n = g.num_vertices();
    const TransitionModel tm{TransitionModel::Kind::uniform_fanout, make_fanouts(fan, L)};
    const VipScores s = propagate(g, tm, std::vector<double>(p0, p0 + n));  // vip.cpp:37
    if (hop_out)
      for (std::uint32_t h = 0; h < L; ++h) std::memcpy(hop_out + h * n, s.hop[h].data(), n * 8);
    std::memcpy(total_out, s.total.data(), n * 8);
  });
}

int ref_empirical_vip(void* gp, const std::uint8_t* roles, const std::uint32_t* labels,
                      std::uint32_t K, std::uint32_t k, std::uint64_t b, const std::uint32_t* fan,
                      std::uint32_t L, std::uint64_t S, std::uint64_t seed, double* out) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const std::uint64_t n = g.num_vertices();
    const auto f = empirical_vip(g, make_roles_view(roles, n), make_part(labels, n, K), k, b,
                                 make_fanouts(fan, L), S, SeedSpec{seed});  // vip.cpp:85
    std::memcpy(out, f.data(), n * 8);
  });
}

// ---- policies ----
int ref_rank_by_scores(const std::uint32_t* labels, std::uint64_t n, std::uint32_t K,
                       std::uint32_t k, const double* scores, std::uint64_t n_scores,
                       std::uint32_t* order_out, double* score_out, std::uint64_t* count) {
  return guard([&] {
    const Ranking r =
        rank_by_scores(make_part(labels, n, K), k, std::span<const double>(scores, n_scores));  // policies.cpp:134
    std::memcpy(order_out, r.order.data(), r.order.size() * 4);
    std::memcpy(score_out, r.score.data(), r.score.size() * 8);
    *count = r.order.size();
  });
}

// build_cache (policies.cpp:149-163) over K rankings given as concatenated
// orders. Writes the per-partition cached prefix lengths and the bitsets.
int ref_build_cache(const std::uint32_t* orders, const std::uint64_t* order_offsets,
                    std::uint32_t K, double alpha, std::uint64_t n, std::uint64_t* take_out,
                    std::uint64_t* bits_out /* K * ((n+63)/64) */) {
  return guard([&] {
    std::vector<Ranking> rk(K);
    for (std::uint32_t k = 0; k < K; ++k) {
      rk[k].partition = k;
      rk[k].order.assign(orders + order_offsets[k], orders + order_offsets[k + 1]);
    }
    const CachePlan plan = build_cache(rk, alpha, n);
    const std::uint64_t W = (n + 63) / 64;
    for (std::uint32_t k = 0; k < K; ++k) {
      take_out[k] = plan.cached[k].size();
      std::memcpy(bits_out + k * W, plan.member_bits[k].data(), W * 8);
    }
  });
}

// simulate (commsim.cpp:77-127) with a plan rebuilt from per-partition
// cached id lists; cells_out is E*K*3 (local, cache, miss), epoch-major.
// simulate with SimulateOptions' trace / batch_costs streams written to
// files (commsim.cpp:104-118) and the optional GPU-prefix split.
int ref_simulate_streams(void* gp, const std::uint8_t* roles, const std::uint32_t* labels, std::uint32_t K,
                         const std::uint32_t* fan, std::uint32_t L, std::uint64_t b, std::uint64_t E,
                         std::uint64_t seed, const std::uint32_t* cached, const std::uint64_t* cached_off,
                         const char* trace_path, const char* costs_path, const std::uint32_t* orderings,
                         const std::uint64_t* ordering_off, double gamma, std::uint64_t* cells_out) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const std::uint64_t n = g.num_vertices();
    CachePlan plan = CachePlan::empty(K, n);
    for (std::uint32_t k = 0; k < K; ++k)
      for (std::uint64_t i = cached_off[k]; i < cached_off[k + 1]; ++i) {
        plan.cached[k].push_back(cached[i]);
        plan.member_bits[k][cached[i] >> 6] |= 1ull << (cached[i] & 63);
      }
    std::ofstream tr, bc;
    SimulateOptions opts;
    if (trace_path) {
      tr.open(trace_path);
      opts.trace = &tr;
    }
    if (costs_path) {
      bc.open(costs_path);
      opts.batch_costs = &bc;
    }
    std::vector<std::vector<vertex_t>> ords;
    if (orderings) {
      for (std::uint32_t k = 0; k < K; ++k) ords.emplace_back(orderings + ordering_off[k], orderings + ordering_off[k + 1]);
      opts.gpu_orderings = &ords;
      opts.gamma = gamma;
    }
    const CommReport r = simulate(g, make_roles_view(roles, n), make_part(labels, n, K), make_fanouts(fan, L), b, E,
                                  SeedSpec{seed}, plan, opts);
    for (std::size_t c = 0; c < r.cells.size(); ++c) {
      cells_out[3 * c] = r.cells[c].local_hits;
      cells_out[3 * c + 1] = r.cells[c].cache_hits;
      cells_out[3 * c + 2] = r.cells[c].remote_misses;
    }
  });
}

int ref_simulate(void* gp, const std::uint8_t* roles, const std::uint32_t* labels, std::uint32_t K,
                 const std::uint32_t* fan, std::uint32_t L, std::uint64_t b, std::uint64_t E,
                 std::uint64_t seed, const std::uint32_t* cached, const std::uint64_t* cached_off,
                 std::uint64_t* cells_out, const std::uint32_t* seed_keys) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const std::uint64_t n = g.num_vertices();
    CachePlan plan = CachePlan::empty(K, n);
    for (std::uint32_t k = 0; k < K; ++k)
      for (std::uint64_t i = cached_off[k]; i < cached_off[k + 1]; ++i) {
        plan.cached[k].push_back(cached[i]);
        plan.member_bits[k][cached[i] >> 6] |= 1ull << (cached[i] & 63);
      }
    std::vector<vertex_t> keys;
    SimulateOptions opts;
    if (seed_keys) {
      keys.assign(seed_keys, seed_keys + n);
      opts.seed_keys = &keys;  // commsim.hpp:44
    }
    const CommReport r = simulate(g, make_roles_view(roles, n), make_part(labels, n, K),
                                  make_fanouts(fan, L), b, E, SeedSpec{seed}, plan, opts);
    for (std::uint64_t e = 0; e < E; ++e)
      for (std::uint32_t k = 0; k < K; ++k) {
        const auto& c = r.at(e, k);
        cells_out[(e * K + k) * 3 + 0] = c.local_hits;
        cells_out[(e * K + k) * 3 + 1] = c.cache_hits;
        cells_out[(e * K + k) * 3 + 2] = c.remote_misses;
      }
  });
}

// Baseline rankings (policies.cpp:57-132). which: 0 degree (L), 1 halo,
// 2 wpr (TransitionModel{f1}, iters, damping), 3 numpaths (L).
int ref_rank_policy(void* gp, int which, const std::uint8_t* roles, const std::uint32_t* labels, std::uint32_t K,
                    std::uint32_t k, std::uint64_t L, std::uint32_t f1, std::uint32_t iters, double damping,
                    std::uint32_t* order, double* score, std::uint64_t* count, double* eff_alpha) {
  return guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const std::uint64_t n = g.num_vertices();
    const PartitionMap part = make_part(labels, n, K);
    const VertexRoles r = make_roles_view(roles, n);
    Ranking rk;
    if (which == 0) rk = rank_degree(g, r, part, k, L);
    else if (which == 1) rk = rank_halo_1hop(g, part, k);
    else if (which == 2)
      rk = rank_wpr(g, r, part, k, TransitionModel{TransitionModel::Kind::uniform_fanout, FanoutSpec{{f1}}}, iters,
                    damping);
    else rk = rank_numpaths(g, r, part, k, L);
    std::memcpy(order, rk.order.data(), rk.order.size() * 4);
    std::memcpy(score, rk.score.data(), rk.score.size() * 8);
    *count = rk.order.size();
    *eff_alpha = rk.effective_alpha;
  });
}

// ---- reorder ----
int ref_build_reorder(const std::uint32_t* labels, std::uint64_t n, std::uint32_t K,
                      const double* scores /* K*n */, std::uint32_t* old_of_new,
                      std::uint64_t* ranges /* 2K */) {
  return guard([&] {
    std::vector<std::vector<double>> s(K);
    for (std::uint32_t k = 0; k < K; ++k) s[k].assign(scores + k * n, scores + (k + 1) * n);
    const ReorderMap map = build_reorder(make_part(labels, n, K), s);  // reorder.cpp:11
    std::memcpy(old_of_new, map.old_of_new.data(), n * 4);
    for (std::uint32_t k = 0; k < K; ++k) {
      ranges[2 * k] = map.ranges[k].first;
      ranges[2 * k + 1] = map.ranges[k].second;
    }
  });
}

// apply_reorder (reorder.cpp:36-70): the relabelled graph (a new handle),
// roles and labels. The map's ranges are not consulted by apply_reorder.
void* ref_apply_reorder(void* gp, const std::uint8_t* roles, const std::uint32_t* labels, std::uint32_t K,
                        const std::uint32_t* old_of_new, std::uint8_t* roles_out, std::uint32_t* labels_out) {
  Graph* out = nullptr;
  const int rc = guard([&] {
    const Graph& g = *static_cast<Graph*>(gp);
    const std::size_t n = g.num_vertices();
    ReorderMap map;
    map.old_of_new.assign(old_of_new, old_of_new + n);
    map.new_of_old.resize(n);
    for (std::size_t i = 0; i < n; ++i) map.new_of_old[map.old_of_new[i]] = static_cast<vertex_t>(i);
    ReorderedDataset d = apply_reorder(g, make_roles_view(roles, n), make_part(labels, n, K), map);
    std::memcpy(roles_out, d.roles.role.data(), n);
    std::memcpy(labels_out, d.part.part_of.data(), n * 4);
    out = new Graph(std::move(d.graph));
  });
  return rc == 0 ? out : nullptr;
}

// ---- rng ----
std::uint64_t ref_mix64(std::uint64_t x) { return mix64(x); }
// SeedSpec::key (rng.hpp:63-67) for tuples of 1..6 parts.
std::uint64_t ref_seed_key(std::uint64_t seed, const std::uint64_t* p, std::uint32_t np) {
  const SeedSpec s{seed};
  switch (np) {
    case 1: return s.key({p[0]});
    case 2: return s.key({p[0], p[1]});
    case 3: return s.key({p[0], p[1], p[2]});
    case 4: return s.key({p[0], p[1], p[2], p[3]});
    case 5: return s.key({p[0], p[1], p[2], p[3], p[4]});
    case 6: return s.key({p[0], p[1], p[2], p[3], p[4], p[5]});
    default: return s.key({});
  }
}
void ref_stream_draws(std::uint64_t key, std::uint64_t bound, std::uint64_t count,
                      std::uint64_t* out) {
  RngStream s(key);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = bound ? s.next_below(bound) : s.next_u64();
}

}  // extern "C"
