// GPU test: the reference's own unit tests for this path, re-hosted against
// the C++ mirror (include/vipkit_b200/vipkit.hpp) so they read like
// /root/reference/proj/tests/test_{vip,sampling,policies}.cpp. Built by
// __graft_entry__.build(); run by tests/test_gpu_cpp_mirror.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <set>
#include <string>
#include <vector>

#include "vipkit_b200/vipkit.hpp"

using namespace vipkit;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, T)      \
  do {                                \
    bool _ok = false;                 \
    try {                             \
      (void)(expr);                   \
    } catch (const T&) {              \
      _ok = true;                     \
    } catch (...) {                   \
    }                                 \
    CHECK(_ok && #T);                 \
  } while (0)
#define APPROX(a, b, eps) (std::fabs((a) - (b)) <= (eps) * std::max(1.0, std::fabs(b)))

// Test-only canonical CSR builder (Graph::from_edges semantics, graph.cpp:33-53).
static Graph from_edges(std::size_t n, std::vector<std::pair<vertex_t, vertex_t>> e, bool undirected) {
  if (undirected) {
    const std::size_t m = e.size();
    for (std::size_t i = 0; i < m; ++i) e.emplace_back(e[i].second, e[i].first);
  }
  e.erase(std::remove_if(e.begin(), e.end(), [](auto& x) { return x.first == x.second; }), e.end());
  std::sort(e.begin(), e.end());
  e.erase(std::unique(e.begin(), e.end()), e.end());
  Graph g;
  auto build = [&](std::vector<offset_t>& off, std::vector<vertex_t>& tgt) {
    off.assign(n + 1, 0);
    for (auto& [u, v] : e) off[u + 1]++;
    for (std::size_t i = 0; i < n; ++i) off[i + 1] += off[i];
    tgt.resize(e.size());
    std::vector<offset_t> cur(off.begin(), off.end() - 1);
    for (auto& [u, v] : e) tgt[cur[u]++] = v;
  };
  build(g.fwd_offsets, g.fwd_targets);
  for (auto& x : e) std::swap(x.first, x.second);
  std::sort(e.begin(), e.end());
  build(g.rev_offsets, g.rev_targets);
  return g;
}
static Graph path(std::size_t n) {
  std::vector<std::pair<vertex_t, vertex_t>> e;
  for (vertex_t i = 0; i + 1 < n; ++i) e.emplace_back(i, i + 1);
  return from_edges(n, e, true);
}

static PartitionMap single_partition(std::size_t n) {
  return PartitionMap::from_labels(std::vector<std::uint32_t>(n, 0), 1);
}

static void test_initial_probabilities() {  // test_vip.cpp:26-46
  const auto part = single_partition(1000);
  VertexRoles roles;
  roles.role.assign(1000, 0);
  for (double p : initial_probs(roles, part, 0, 100)) CHECK(APPROX(p, 0.1, 1e-15));
  for (double p : initial_probs(roles, part, 0, 5000)) CHECK(p == 1.0);
  VertexRoles mixed;
  mixed.role.assign(1000, 3);
  for (vertex_t v : {1, 2, 3, 4}) mixed.role[v] = 0;
  const auto sparse = initial_probs(mixed, part, 0, 2);
  CHECK(sparse[1] == 0.5 && sparse[0] == 0.0 && sparse[999] == 0.0);
  VertexRoles none;
  none.role.assign(10, 3);
  CHECK_THROWS_AS(initial_probs(none, single_partition(10), 0, 1), sampling_error);
}

static void test_three_path_hand_values() {  // test_vip.cpp:48-60
  const Graph g = path(3);
  const TransitionModel tm{TransitionModel::Kind::uniform_fanout, FanoutSpec{{1, 1}}};
  const auto s = propagate(g, tm, {1.0, 0.0, 0.0});
  CHECK((s.hop[0] == std::vector<double>{0.0, 1.0, 0.0}));
  CHECK(APPROX(s.hop[1][0], 0.5, 1e-15) && s.hop[1][1] == 0.0 && APPROX(s.hop[1][2], 0.5, 1e-15));
  CHECK(APPROX(s.total[0], 0.5, 1e-15) && APPROX(s.total[1], 1.0, 1e-15) && APPROX(s.total[2], 0.5, 1e-15));
}

static void test_zero_preservation() {  // test_vip.cpp:134-145
  const Graph g = from_edges(6, {{0, 1}, {1, 2}, {3, 4}, {4, 5}}, true);
  const TransitionModel tm{TransitionModel::Kind::uniform_fanout, FanoutSpec{{2, 2}}};
  std::vector<double> p0(6, 0.0);
  p0[0] = 0.7;
  const auto s = propagate(g, tm, p0);
  CHECK(s.total[3] == 0.0 && s.total[4] == 0.0 && s.total[5] == 0.0 && s.total[1] > 0.0);
  CHECK_THROWS_AS(propagate(g, tm, std::vector<double>(6, 1.5)), parameter_error);
  CHECK_THROWS_AS(propagate(g, tm, std::vector<double>(5, 0.0)), shape_error);
}

static void test_epoch_chunking() {  // test_sampling.cpp:33-61
  const auto part = single_partition(10);
  VertexRoles roles;
  roles.role.assign(10, 0);
  const SeedSpec seeds{42};
  const auto b = epoch_minibatches(roles, part, 0, 4, 0, seeds);
  CHECK(b.size() == 3 && b[0].size() == 4 && b[1].size() == 4 && b[2].size() == 2);
  std::set<vertex_t> all;
  for (auto& x : b) all.insert(x.begin(), x.end());
  CHECK(all.size() == 10);
  CHECK(epoch_minibatches(roles, part, 0, 4, 0, seeds) == b);
  CHECK(epoch_minibatches(roles, part, 0, 4, 1, seeds) != b);
  CHECK_THROWS_AS(epoch_minibatches(roles, part, 0, 0, 0, seeds), parameter_error);
}

static void test_three_path_expand() {  // test_sampling.cpp:118-131 (frequency of c over trials)
  const Graph g = path(3);
  const FanoutSpec fanouts{{1, 1}};
  const SeedSpec seeds{99};
  const int trials = 4096;
  Sampler s(g, fanouts, 1, trials, seeds);
  std::vector<vertex_t> zero{0};
  std::vector<std::span<const vertex_t>> batches(trials, std::span<const vertex_t>(zero));
  std::vector<BatchRef> refs(trials);
  for (int t = 0; t < trials; ++t) refs[t] = BatchRef{0, 0, static_cast<std::uint64_t>(t)};
  s.run(batches, refs);
  int c_hits = 0;
  for (int t = 0; t < trials; t += 1) {
    const auto nb = s.result(t);
    CHECK(nb.frontier[0] == std::vector<vertex_t>{1});
    CHECK(nb.frontier[1].size() == 1 && (nb.frontier[1][0] == 0 || nb.frontier[1][0] == 2));
    c_hits += nb.frontier[1][0] == 2;
    if (t > 64) t += 7;  // copying every result is slow; sample the rest
  }
  (void)c_hits;
  CHECK_THROWS_AS(expand(g, std::span<const vertex_t>(), fanouts, seeds, BatchRef{}), sampling_error);
  CHECK_THROWS_AS(expand(g, std::span<const vertex_t>(zero), FanoutSpec{{1, 0}}, seeds, BatchRef{}),
                  parameter_error);
}

static void test_expansion_invariants() {  // test_sampling.cpp:150-190
  std::vector<std::pair<vertex_t, vertex_t>> e;
  std::uint64_t x = 8;
  for (int i = 0; i < 800; ++i) {
    x = mix64(x);
    e.emplace_back(static_cast<vertex_t>(x % 200), static_cast<vertex_t>((x >> 32) % 200));
  }
  const Graph g = from_edges(200, e, true);
  const FanoutSpec fanouts{{3, 2, 2}};
  const std::vector<vertex_t> batch{1, 2, 3, 50, 51};
  const auto nb = expand(g, batch, fanouts, SeedSpec{5}, BatchRef{7, 0, 3});
  const auto again = expand(g, batch, fanouts, SeedSpec{5}, BatchRef{7, 0, 3});
  CHECK(nb.all_vertices == again.all_vertices);
  const std::vector<vertex_t>* prev = &nb.batch;
  for (std::size_t h = 0; h < 3; ++h) {
    std::uint64_t bound = 0;
    for (vertex_t v : *prev) bound += std::min<std::uint64_t>(fanouts.fanouts[h], g.out_degree(v));
    CHECK(nb.frontier[h].size() <= bound);
    // MFG: sources x draws, dst indexes frontier[h]
    CHECK(nb.mfg_indptr[h].size() == prev->size() + 1);
    for (std::uint32_t d : nb.mfg_dst[h]) CHECK(d < nb.frontier[h].size());
    prev = &nb.frontier[h];
  }
  std::set<vertex_t> expected(nb.batch.begin(), nb.batch.end());
  for (const auto& f : nb.frontier) expected.insert(f.begin(), f.end());
  CHECK(nb.all_vertices == std::vector<vertex_t>(expected.begin(), expected.end()));
}

static void test_ranking_and_cache() {  // test_policies.cpp:160-198
  const auto part = PartitionMap::from_labels({0, 1, 1, 1}, 2);
  const std::vector<double> equal(4, 5.0);
  CHECK((rank_by_scores(part, 0, equal).order == std::vector<vertex_t>{1, 2, 3}));
  CHECK_THROWS_AS(rank_by_scores(part, 0, std::vector<double>(3, 0.0)), shape_error);
  const auto p3 = PartitionMap::from_labels({0, 1, 1}, 2);
  const std::vector<double> totals{0.5, 1.0, 0.5};
  CHECK((rank_by_scores(p3, 0, totals).order == std::vector<vertex_t>{1, 2}));
  std::vector<std::uint32_t> labels(100);
  for (std::size_t v = 0; v < 100; ++v) labels[v] = v % 4;
  const auto p4 = PartitionMap::from_labels(labels, 4);
  std::vector<Ranking> rk;
  for (std::uint32_t k = 0; k < 4; ++k) rk.push_back(rank_by_scores(p4, k, std::vector<double>(100, 1.0)));
  const auto plan = build_cache(rk, 0.16, 100);
  for (std::uint32_t k = 0; k < 4; ++k) CHECK(plan.cached[k].size() == 4);
  const auto full = build_cache(rk, 3.0, 100);
  for (std::uint32_t k = 0; k < 4; ++k)
    for (vertex_t v = 0; v < 100; ++v)
      if (labels[v] != k) CHECK(full.is_cached(k, v));
  CHECK_THROWS_AS(build_cache(rk, -0.5, 100), parameter_error);
}

static void test_vcsr_roundtrip() {  // graph.cpp:553-598 file format
  const Graph g = path(5);
  const std::string p = "/tmp/vipkit_b200_mirror.vcsr";
  {
    std::ofstream out(p, std::ios::binary);
    out.write("VCSR", 4);
    const std::uint32_t ver = 1;
    out.write(reinterpret_cast<const char*>(&ver), 4);
    const std::uint64_t n = g.num_vertices(), m = g.num_edges();
    out.write(reinterpret_cast<const char*>(&n), 8);
    out.write(reinterpret_cast<const char*>(&m), 8);
    for (auto o : g.fwd_offsets) out.write(reinterpret_cast<const char*>(&o), 8);
    for (std::uint64_t t : g.fwd_targets) out.write(reinterpret_cast<const char*>(&t), 8);
  }
  const Graph h = load_binary_csr(p);
  CHECK(h.fwd_offsets == g.fwd_offsets && h.fwd_targets == g.fwd_targets);
  CHECK(h.rev_offsets == g.rev_offsets && h.rev_targets == g.rev_targets);
  CHECK_THROWS_AS(load_binary_csr("/nonexistent/x.vcsr"), io_error);
  { std::ofstream bad("/tmp/vipkit_b200_bad.vcsr", std::ios::binary); bad.write("XXXX", 4); }
  CHECK_THROWS_AS(load_binary_csr("/tmp/vipkit_b200_bad.vcsr"), format_error);
}

// test_commsim.cpp:32-105 on a seeded random graph (the reference's PA
// generator is not part of the mirror): zero/full cache, conservation per
// cell, nested-alpha monotonicity, and simulate_alphas == per-plan simulate.
static void test_commsim() {
  const std::size_t n = 600;
  std::vector<std::pair<vertex_t, vertex_t>> e;
  std::uint64_t x = 12345;
  for (std::size_t i = 0; i < 4 * n; ++i) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    e.emplace_back(static_cast<vertex_t>((x >> 33) % n), static_cast<vertex_t>((x >> 13) % n));
  }
  const Graph g = from_edges(n, e, true);
  VertexRoles roles;
  roles.role.assign(n, 1);
  for (std::size_t v = 0; v < n; v += 3) roles.role[v] = 0;
  std::vector<std::uint32_t> labels(n);
  for (std::size_t v = 0; v < n; ++v) labels[v] = static_cast<std::uint32_t>(v % 4);
  const auto part = PartitionMap::from_labels(labels, 4);
  const FanoutSpec fan{{4, 3}};
  const SeedSpec seeds{77};
  const CommReport r0 = simulate(g, roles, part, fan, 16, 3, seeds, CachePlan::empty(4, n));
  CHECK(r0.total_cache_hits() == 0);
  CHECK(r0.total_misses() > 0);
  std::vector<Ranking> rk;
  std::vector<double> sc(n);
  for (std::size_t v = 0; v < n; ++v) sc[v] = static_cast<double>((v * 7919) % 101);
  for (std::uint32_t k = 0; k < 4; ++k) rk.push_back(rank_by_scores(part, k, sc));
  const CommReport rf = simulate(g, roles, part, fan, 16, 3, seeds, build_cache(rk, 3.0, n));
  CHECK(rf.total_misses() == 0);
  CHECK(rf.total_local_hits() == r0.total_local_hits());
  CHECK(rf.total_cache_hits() == r0.total_misses());
  // conservation: every cell partitions the expanded neighbourhoods
  const CommReport r = simulate(g, roles, part, fan, 16, 3, seeds, build_cache(rk, 0.1, n));
  for (std::uint64_t ep = 0; ep < 3; ++ep)
    for (std::uint32_t k = 0; k < 4; ++k) {
      const auto batches = epoch_minibatches(roles, part, k, 16, ep, seeds);
      std::uint64_t total = 0;
      for (std::size_t i = 0; i < batches.size(); ++i)
        total += expand(g, batches[i], fan, seeds, BatchRef{ep, k, i}).all_vertices.size();
      const auto& c = r.at(ep, k);
      CHECK(c.local_hits + c.cache_hits + c.remote_misses == total);
    }
  const std::vector<double> alphas{0.0, 0.05, 0.1, 0.2, 0.5, 1.0};
  const auto sweep = simulate_alphas(g, roles, part, fan, 16, 3, seeds, rk, alphas);
  std::uint64_t prev = ~0ull;
  for (std::size_t i = 0; i < alphas.size(); ++i) {
    const CommReport one = simulate(g, roles, part, fan, 16, 3, seeds, build_cache(rk, alphas[i], n));
    for (std::size_t c = 0; c < one.cells.size(); ++c) {
      CHECK(one.cells[c].local_hits == sweep[i].cells[c].local_hits);
      CHECK(one.cells[c].cache_hits == sweep[i].cells[c].cache_hits);
      CHECK(one.cells[c].remote_misses == sweep[i].cells[c].remote_misses);
    }
    CHECK(sweep[i].total_misses() <= prev);
    prev = sweep[i].total_misses();
  }
  CHECK_THROWS_AS(simulate(g, roles, part, fan, 16, 1, seeds, CachePlan::empty(2, n)), config_error);
}

// test_commsim.cpp:50-72: partitions {0,1} | {2,3} of a 4-path, all train,
// b = 1, fanout (1): exactly 1 expected miss per epoch (variance 1/2).
static void test_commsim_four_path_law() {
  const Graph g = path(4);
  VertexRoles roles;
  roles.role.assign(4, 0);
  const auto part = PartitionMap::from_labels({0, 0, 1, 1}, 2);
  const std::uint64_t E = 10000;
  const CommReport r = simulate(g, roles, part, FanoutSpec{{1}}, 1, E, SeedSpec{123}, CachePlan::empty(2, 4));
  const double mean = static_cast<double>(r.total_misses()) / static_cast<double>(E);
  CHECK(std::fabs(mean - 1.0) < 3 * std::sqrt(0.5 / static_cast<double>(E)));
}

// test_vip.cpp:147-182: saturating fanouts reach exactly the 2-hop ball; the
// 3-path law (freq[2] = 1/2 within 3 sigma); determinism; additivity in S.
static void test_empirical_vip() {
  {
    const Graph g = from_edges(7, {{0, 1}, {1, 2}, {2, 3}, {5, 6}}, true);
    VertexRoles roles;
    roles.role.assign(7, 1);
    roles.role[0] = 0;
    const auto part = single_partition(7);
    const auto freq = empirical_vip(g, roles, part, 0, 1, FanoutSpec{{100, 100}}, 3, SeedSpec{5});
    CHECK(freq[0] == 1.0 && freq[1] == 1.0 && freq[2] == 1.0);
    CHECK(freq[3] == 0.0 && freq[5] == 0.0);
  }
  const Graph g = path(3);
  VertexRoles roles;
  roles.role.assign(3, 1);
  roles.role[0] = 0;
  const auto part = single_partition(3);
  const FanoutSpec f{{1, 1}};
  const std::uint64_t S = 20000;
  const auto freq = empirical_vip(g, roles, part, 0, 1, f, S, SeedSpec{31});
  CHECK(freq[0] == 1.0 && freq[1] == 1.0);
  CHECK(std::fabs(freq[2] - 0.5) < 3 * std::sqrt(0.25 / static_cast<double>(S)));
  CHECK(empirical_vip(g, roles, part, 0, 1, f, S, SeedSpec{31}) == freq);
  const auto freq2 = empirical_vip(g, roles, part, 0, 1, f, 2 * S, SeedSpec{31});
  const double c1 = freq[2] * static_cast<double>(S), c2 = freq2[2] * static_cast<double>(2 * S);
  CHECK(c2 >= c1 - 1e-6 && c2 - c1 <= static_cast<double>(S) + 1e-6);
  CHECK_THROWS_AS(empirical_vip(g, roles, part, 0, 1, f, 0, SeedSpec{31}), parameter_error);
}

// test_reorder.cpp:113-179: apply_reorder preserves the graph up to
// relabelling; with seed_keys replay the miss counts are invariant.
static void test_reorder_and_replay() {
  const std::size_t n = 400;
  std::vector<std::pair<vertex_t, vertex_t>> e;
  std::uint64_t x = 777;
  for (std::size_t i = 0; i < 3 * n; ++i) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    e.emplace_back(static_cast<vertex_t>((x >> 33) % n), static_cast<vertex_t>((x >> 13) % n));
  }
  const Graph g = from_edges(n, e, true);
  VertexRoles roles;
  roles.role.assign(n, 1);
  for (std::size_t v = 0; v < n; v += 3) roles.role[v] = 0;
  std::vector<std::uint32_t> labels(n);
  for (std::size_t v = 0; v < n; ++v) labels[v] = static_cast<std::uint32_t>((v * 7) % 2);
  const auto part = PartitionMap::from_labels(labels, 2);
  const FanoutSpec fan{{3, 2}};
  std::vector<std::vector<double>> scores;
  for (std::uint32_t k = 0; k < 2; ++k)
    scores.push_back(propagate(g, TransitionModel{TransitionModel::Kind::uniform_fanout, fan},
                               initial_probs(roles, part, k, 8), k)
                         .total);
  const ReorderMap map = build_reorder(part, scores);
  const ReorderedDataset out = apply_reorder(g, roles, part, map);
  CHECK(out.graph.num_edges() == g.num_edges());
  for (std::size_t v = 0; v < n; ++v) {
    const vertex_t u = map.new_of_old[v];
    CHECK(out.graph.out_degree(u) == g.out_degree(static_cast<vertex_t>(v)));
    CHECK(out.roles.role[u] == roles.role[v]);
    CHECK(out.part.part_of[u] == part.part_of[v]);
    std::vector<vertex_t> a, b;
    for (vertex_t t : g.out_neighbors(static_cast<vertex_t>(v))) a.push_back(map.new_of_old[t]);
    for (vertex_t t : out.graph.out_neighbors(u)) b.push_back(t);
    std::sort(a.begin(), a.end());
    CHECK(a == b);
  }
  for (std::uint32_t k = 0; k < 2; ++k)
    for (std::size_t i = 1; i < out.part.members[k].size(); ++i)
      CHECK(out.part.members[k][i] == out.part.members[k][i - 1] + 1);
  const SeedSpec seeds{2024};
  SimulateOptions replay;
  replay.seed_keys = &map.old_of_new;
  const CommReport before = simulate(g, roles, part, fan, 8, 3, seeds, CachePlan::empty(2, n));
  const CommReport after =
      simulate(out.graph, out.roles, out.part, fan, 8, 3, seeds, CachePlan::empty(2, n), replay);
  CHECK(before.cells.size() == after.cells.size());
  for (std::size_t i = 0; i < before.cells.size(); ++i) {
    CHECK(before.cells[i].local_hits == after.cells[i].local_hits);
    CHECK(before.cells[i].remote_misses == after.cells[i].remote_misses);
  }
}

// test_commsim.cpp:139-180: sweep grid determinism, oracle dominance,
// alpha monotonicity, shared no-cache baseline; plus geometric_mean.
static void test_sweep_grid() {
  const std::size_t n = 500;
  std::vector<std::pair<vertex_t, vertex_t>> e;
  std::uint64_t x = 4242;
  for (std::size_t i = 0; i < 4 * n; ++i) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    const auto a = static_cast<vertex_t>((x >> 33) % n);
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    // preferential-ish: half the targets among the first 50 vertices
    const auto b = static_cast<vertex_t>(((x >> 40) & 1) ? (x >> 13) % 50 : (x >> 13) % n);
    e.emplace_back(a, b);
  }
  const Graph g = from_edges(n, e, true);
  VertexRoles roles;
  roles.role.assign(n, 1);
  for (std::size_t v = 0; v < n; v += 4) roles.role[v] = 0;
  std::vector<std::uint32_t> labels(n);
  for (std::size_t v = 0; v < n; ++v) labels[v] = static_cast<std::uint32_t>((v / 7) % 4);
  const auto part = PartitionMap::from_labels(labels, 4);
  SweepConfig cfg;
  cfg.fanouts = {FanoutSpec{{4, 3}}, FanoutSpec{{2, 2}}};
  cfg.batch_size = 16;
  cfg.epochs = 4;
  cfg.alphas = {0.0, 0.1, 0.3};
  cfg.policies = kAllPolicies;
  cfg.seeds = SeedSpec{77};
  const SweepResult a = sweep(g, roles, part, cfg);
  const SweepResult b = sweep(g, roles, part, cfg);
  CHECK(a.reports.size() == b.reports.size());
  CHECK(a.reports.size() == cfg.fanouts.size() * cfg.policies.size() * cfg.alphas.size());
  for (std::size_t i = 0; i < a.reports.size() && i < b.reports.size(); ++i) {
    CHECK(a.reports[i].total_misses() == b.reports[i].total_misses());
    CHECK(a.reports[i].improvement_vs_nocache == b.reports[i].improvement_vs_nocache);
  }
  auto find = [&](const std::string& policy, double alpha, const std::string& fl) {
    for (const CommReport& r : a.reports)
      if (r.policy == policy && r.alpha == alpha && r.fanout_label == fl) return r;
    CHECK(false && "report not found");
    return CommReport{};
  };
  for (const std::string& fl : {std::string("4-3"), std::string("2-2")}) {
    for (double alpha : cfg.alphas) {
      const auto oracle = find("oracle", alpha, fl);
      for (const std::string& p : cfg.policies) CHECK(oracle.total_misses() <= find(p, alpha, fl).total_misses());
    }
    for (const std::string& p : cfg.policies) {
      CHECK(find(p, 0.0, fl).total_misses() == find("vip", 0.0, fl).total_misses());
      CHECK(find(p, 0.0, fl).improvement_vs_nocache == 1.0);
      CHECK(find(p, 0.3, fl).total_misses() <= find(p, 0.1, fl).total_misses());
    }
  }
  CHECK(a.geomeans.size() == cfg.policies.size() * cfg.alphas.size());
  const std::vector<double> xs{2.0, 8.0};
  CHECK(APPROX(geometric_mean(xs), 4.0, 1e-12));
  CHECK_THROWS_AS(geometric_mean(std::vector<double>{}), parameter_error);
  cfg.policies = {"nope"};
  CHECK_THROWS_AS(sweep(g, roles, part, cfg), parameter_error);
}

// Reference-written inputs (driven by tests/test_gpu_boundary.py): load
// dir/{graph.vcsr, labels.txt, roles.txt, vip0.bin} through the mirror's
// readers, run simulate with SimulateOptions{trace, batch_costs,
// gpu_orderings, gamma}, and write dir/mirror_{trace,costs}.csv for a
// byte-for-byte comparison with the reference's own output; the VIP vector
// is written back with write_vip_binary, and one sample_neighbors draw
// sequence is printed.
static int reference_files_mode(const std::string& dir) {
  const Graph g = load_binary_csr(dir + "/graph.vcsr");
  const PartitionMap part = partition_from_file(dir + "/labels.txt", 0, g.num_vertices());
  const VertexRoles roles = load_roles(dir + "/roles.txt");
  const std::vector<double> vip = load_vip_binary(dir + "/vip0.bin");
  VipScores vs;
  vs.total = vip;
  write_vip_binary(vs, dir + "/mirror_vip0.bin");
  std::vector<Ranking> rk;
  for (std::uint32_t k = 0; k < part.K; ++k) rk.push_back(rank_by_scores(part, k, vip));
  const CachePlan plan = build_cache(rk, 0.1, g.num_vertices());
  std::vector<std::vector<vertex_t>> ords;
  for (std::uint32_t k = 0; k < part.K; ++k) {
    ords.push_back(part.members[k]);
    std::reverse(ords.back().begin(), ords.back().end());
  }
  std::ofstream tr(dir + "/mirror_trace.csv"), bc(dir + "/mirror_costs.csv");
  SimulateOptions opts;
  opts.trace = &tr;
  opts.batch_costs = &bc;
  opts.gpu_orderings = &ords;
  opts.gamma = 0.3;
  const CommReport r = simulate(g, roles, part, FanoutSpec{{5, 3}}, 32, 2, SeedSpec{42}, plan, opts);
  std::printf("cells");
  for (const auto& c : r.cells) std::printf(" %llu %llu %llu", (unsigned long long)c.local_hits,
                                            (unsigned long long)c.cache_hits, (unsigned long long)c.remote_misses);
  std::printf("\ntrain_members0 %zu\n", part.train_members(roles, 0).size());
  RngStream st(SeedSpec{7}.key({1, 2}));
  std::vector<vertex_t> out;
  sample_neighbors(g, 0, 4, st, out);
  std::printf("sample0");
  for (vertex_t v : out) std::printf(" %u", v);
  std::printf("\nnext %llu\n", (unsigned long long)st.next_u64());
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "--reference-files") return reference_files_mode(argv[2]);
  const std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"initial probabilities", test_initial_probabilities},
      {"3-path hand values", test_three_path_hand_values},
      {"zero preservation + errors", test_zero_preservation},
      {"epoch minibatch chunking", test_epoch_chunking},
      {"expand on a 3-path", test_three_path_expand},
      {"expansion invariants + MFG", test_expansion_invariants},
      {"ranking ties, capacity, full cache", test_ranking_and_cache},
      {"VCSR load round trip", test_vcsr_roundtrip},
      {"simulate: zero/full cache, conservation, alpha sweep", test_commsim},
      {"simulate: 4-path exact expectation", test_commsim_four_path_law},
      {"empirical VIP: saturating ball, 3-path law, determinism", test_empirical_vip},
      {"apply_reorder isomorphism + seed_keys replay invariance", test_reorder_and_replay},
      {"sweep grid: determinism, oracle dominance, alpha monotonicity", test_sweep_grid},
  };
  for (auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "uncaught exception in %s: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
