"""CPU: the reference's own known-answer tests for this path, re-hosted
against the C restatement (the reference's doctest suites do not build here:
doctest.h is absent). Sources: /root/reference/proj/tests/test_vip.cpp,
test_sampling.cpp, test_policies.cpp, test_commsim.cpp, oracles.hpp."""
import itertools

import numpy as np
import pytest

from oracle.oracle import OracleError


# ---- independent oracles (tests/oracles.hpp:28-119), restated in Python ----
def enumerate_process(g, batch, fanouts):
    """Exact law of the expansion process by exhaustive enumeration
    (oracles.hpp:28-104)."""
    n = g.n
    hop_prob = np.zeros((len(fanouts), n))
    any_prob = np.zeros(n)

    def rec(frontier, h, prob, seen):
        seen = seen | set(frontier)
        if h > len(fanouts):
            for v in seen:
                any_prob[v] += prob
            return
        choices = []
        for v in frontier:
            nb = list(g.tgt[g.off[v]:g.off[v + 1]])
            take = min(fanouts[h - 1], len(nb))
            choices.append([()] if take == 0 else list(itertools.combinations(nb, take)))
        for pick in itertools.product(*choices):
            p = prob
            for c in choices:
                p /= len(c)
            nxt = sorted(set(u for s in pick for u in s))
            for u in nxt:
                hop_prob[h - 1][u] += p
            rec(nxt, h + 1, p, seen)

    rec(list(batch), 1, 1.0, set())
    return hop_prob, any_prob


def walk_reachability(g, src, hops):
    """oracles.hpp:108-119."""
    reach = np.zeros((hops + 1, g.n), bool)
    reach[0, list(src)] = True
    for h in range(1, hops + 1):
        for v in np.nonzero(reach[h - 1])[0]:
            reach[h, g.tgt[g.off[v]:g.off[v + 1]]] = True
    return reach


def binom_3sigma(p, n):
    return 3 * np.sqrt(p * (1 - p) / n)


# ---- test_vip.cpp ----
def test_initial_probs(port):
    """test_vip.cpp:26-46"""
    part = np.zeros(1000, np.uint32)
    roles = np.zeros(1000, np.uint8)
    assert np.allclose(port.initial_probs(roles, part, 1, 0, 100), 0.1, rtol=1e-15)
    assert np.all(port.initial_probs(roles, part, 1, 0, 5000) == 1.0)
    mixed = np.full(1000, 3, np.uint8)
    mixed[[1, 2, 3, 4]] = 0
    p = port.initial_probs(mixed, part, 1, 0, 2)
    assert p[1] == 0.5 and p[0] == 0.0 and p[999] == 0.0
    with pytest.raises(OracleError) as e:
        port.initial_probs(np.full(10, 3, np.uint8), np.zeros(10, np.uint32), 1, 0, 1)
    assert e.value.kind == "sampling_error"


def test_three_path_hand_values(port):
    """test_vip.cpp:48-60"""
    g = port.generate("path", 3)
    hop, tot = port.propagate(g, [1, 1], [1.0, 0.0, 0.0])
    assert list(hop[0]) == [0.0, 1.0, 0.0]
    assert hop[1][0] == pytest.approx(0.5, rel=1e-15) and hop[1][1] == 0.0
    assert hop[1][2] == pytest.approx(0.5, rel=1e-15)
    assert tot == pytest.approx([0.5, 1.0, 0.5], rel=1e-15)


def test_saturating_reachability(port):
    """test_vip.cpp:62-73"""
    g = port.generate("pa", 150, 3, 13)
    p0 = np.zeros(150)
    p0[5] = 1.0
    hop, _ = port.propagate(g, [1000] * 3, p0)
    reach = walk_reachability(g, [5], 3)
    for h in range(1, 4):
        np.testing.assert_array_equal(hop[h - 1], reach[h].astype(float))


def test_directed_tree_exact_law(port):
    """test_vip.cpp:75-95"""
    g = port.from_edges(13, [((v - 1) // 3, v) for v in range(1, 13)], undirected=False)
    p0 = np.zeros(13)
    p0[0] = 1.0
    hop, tot = port.propagate(g, [2, 2], p0)
    law_hop, law_any = enumerate_process(g, [0], [2, 2])
    np.testing.assert_allclose(hop, law_hop, rtol=1e-12, atol=0)
    np.testing.assert_allclose(tot[1:], law_any[1:], rtol=1e-12, atol=0)


def test_monotonicity_and_shared_prefix(port):
    """test_vip.cpp:108-132"""
    g = port.generate("uniform", 300, 4, 77)
    p0 = np.zeros(g.n)
    draws = port.stream_draws(123, 0, 100)
    for i, v in enumerate(range(0, g.n, 3)):
        p0[v] = float(int(draws[i]) >> 11) * 2.0 ** -53
    s_hop, s_tot = port.propagate(g, [2, 3], p0)
    l_hop, l_tot = port.propagate(g, [3, 5], p0)
    d_hop, d_tot = port.propagate(g, [2, 3, 2], p0)
    assert np.all((s_hop >= 0) & (s_hop <= 1))
    assert np.all(s_hop <= l_hop + 1e-15)
    np.testing.assert_array_equal(s_hop, d_hop[:2])
    assert np.all(s_tot <= l_tot + 1e-15) and np.all(s_tot <= d_tot + 1e-15)


def test_zero_preservation(port):
    """test_vip.cpp:134-145"""
    g = port.from_edges(6, [(0, 1), (1, 2), (3, 4), (4, 5)], undirected=True)
    p0 = np.zeros(6)
    p0[0] = 0.7
    _, tot = port.propagate(g, [2, 2], p0)
    assert tot[3] == tot[4] == tot[5] == 0.0 and tot[1] > 0.0


# ---- test_sampling.cpp ----
def test_epoch_chunking(port):
    """test_sampling.cpp:33-61"""
    part = np.zeros(10, np.uint32)
    roles = np.zeros(10, np.uint8)
    b = port.epoch_minibatches(roles, part, 0, 4, 0, 42)
    assert [len(x) for x in b] == [4, 4, 2]
    assert sorted(np.concatenate(b).tolist()) == list(range(10))
    one = port.epoch_minibatches(roles, part, 0, 64, 0, 42)
    assert len(one) == 1 and sorted(one[0].tolist()) == list(range(10))
    b1 = port.epoch_minibatches(roles, part, 0, 4, 1, 42)
    assert any(not np.array_equal(x, y) for x, y in zip(b, b1))
    with pytest.raises(OracleError):
        port.epoch_minibatches(roles, part, 0, 0, 0, 42)
    with pytest.raises(OracleError) as e:
        port.epoch_minibatches(np.full(10, 3, np.uint8), part, 0, 4, 0, 42)
    assert e.value.kind == "sampling_error"


def test_three_path_expand_frequencies(port):
    """test_sampling.cpp:118-131 (3-path, fanout (1,1), c-hit frequency 1/2)."""
    g = port.generate("path", 3)
    trials = 20000
    c_hits = 0
    for t in range(trials):
        x = port.expand(g, [0], [1, 1], 99, 0, 0, t)
        assert list(x.frontier[0]) == [1]
        assert x.frontier[1][0] in (0, 2)
        c_hits += x.frontier[1][0] == 2
    assert abs(c_hits / trials - 0.5) < binom_3sigma(0.5, trials)


def test_saturating_expand_is_l_hop_neighbourhood(port):
    """test_sampling.cpp:118-131"""
    g = port.generate("pa", 120, 3, 5)
    x = port.expand(g, [3, 17], [1000, 1000], 1, 0, 0, 0)
    reach = walk_reachability(g, [3, 17], 2)
    for h in (1, 2):
        np.testing.assert_array_equal(x.frontier[h - 1], np.nonzero(reach[h])[0])


def test_expansion_invariants(port):
    """test_sampling.cpp:150-190"""
    g = port.generate("uniform", 200, 4, 8).ensure_reverse()
    batch = [1, 2, 3, 50, 51]
    x = port.expand(g, batch, [3, 2, 2], 5, 7, 0, 3)
    y = port.expand(g, batch, [3, 2, 2], 5, 7, 0, 3)
    np.testing.assert_array_equal(x.all_vertices, y.all_vertices)
    prev = np.array(batch)
    deg = np.diff(g.off)
    for h, f in enumerate([3, 2, 2]):
        assert len(x.frontier[h]) <= np.minimum(f, deg[prev]).sum()
        for u in x.frontier[h]:
            assert np.isin(g.rev_tgt[g.rev_off[u]:g.rev_off[u + 1]], prev).any()
        prev = x.frontier[h]
    union = np.unique(np.concatenate([batch] + x.frontier))
    np.testing.assert_array_equal(x.all_vertices, union)


# ---- test_policies.cpp / test_commsim.cpp ----
def test_tie_order_and_shape(port):
    """test_policies.cpp:160-173"""
    o, _ = port.rank_by_scores(np.array([0, 1, 1, 1], np.uint32), 2, 0, np.full(4, 5.0))
    assert list(o) == [1, 2, 3]
    with pytest.raises(OracleError) as e:
        port.rank_by_scores(np.array([0, 1, 1, 1], np.uint32), 2, 0, np.zeros(3))
    assert e.value.kind == "shape_error"
    o, _ = port.rank_by_scores(np.array([0, 1, 1], np.uint32), 2, 0, np.array([0.5, 1.0, 0.5]))
    assert list(o) == [1, 2]


def test_capacity_rules(port):
    """test_policies.cpp:175-198: floor(.16*100/4) = 4; alpha >= K-1 caches all remotes."""
    assert port.cache_capacity(0.16, 100, 4) == 4
    assert port.cache_capacity(0.0, 100, 4) == 0
    with pytest.raises(OracleError):
        port.cache_capacity(-0.5, 100, 4)
    labels = (np.arange(100) % 4).astype(np.uint32)
    orders = [port.rank_by_scores(labels, 4, k, np.ones(100))[0] for k in range(4)]
    cached, bits = port.build_cache(orders, 3.0, 100)
    for k in range(4):
        assert len(cached[k]) == 75


def test_two_partition_four_path(port):
    """test_commsim.cpp:50-75: expected misses per epoch is exactly 1."""
    g = port.generate("path", 4)
    roles = np.zeros(4, np.uint8)
    labels = np.array([0, 0, 1, 1], np.uint32)
    exp = 0.0
    for v in range(4):
        _, law_any = enumerate_process(g, [v], [1])
        exp += sum(law_any[u] for u in range(4) if labels[u] != labels[v])
    assert exp == pytest.approx(1.0, abs=1e-12)
    E = 3000
    misses = 0
    for e in range(E):
        for k in range(2):
            for i, b in enumerate(port.epoch_minibatches(roles, labels, k, 1, e, 123)):
                x = port.expand(g, b, [1], 123, e, k, i)
                misses += port.classify(x.all_vertices, labels, k)[2]
    assert abs(misses / E - 1.0) < 3 * np.sqrt(0.5 / E)
