"""CPU: pin the C restatement (oracle/vipkit_port.c) to the reference's own
outputs stored in tests/golden (made by oracle/make_golden.py from the
unmodified reference library). Bit-exact everywhere, including VIP: the port
follows the reference's arithmetic order exactly."""
import numpy as np
import pytest

from conftest import csr_from


def test_rng_golden(port, golden):
    g = golden("rng.npz")
    assert [port.mix64(int(x)) for x in g["xs"]] == [int(x) for x in g["mixes"]]
    keys = [port.seed_key(42, [0xB2, 0, 0, 0, 1, v]) for v in range(16)]
    keys += [port.seed_key(42, [0xB1, 3, 5]), port.seed_key(7, [0xA1, 1])]
    assert keys == [int(x) for x in g["keys"]]
    for i, b in enumerate(g["bounds"]):
        np.testing.assert_array_equal(port.stream_draws(12345 + i, int(b), 64), g["draws"][i])


@pytest.mark.parametrize("name,kind,n,d,s", [
    ("path3", "path", 3, 2, 0), ("star5", "star", 5, 2, 0), ("tree13", "tree", 13, 3, 0),
    ("grid20", "grid", 20, 4, 0), ("pa400", "pa", 400, 4, 15), ("pa150", "pa", 150, 3, 13),
    ("pa120", "pa", 120, 3, 5), ("uni200", "uniform", 200, 4, 8), ("uni300", "uniform", 300, 4, 77),
    ("pa5000", "pa", 5000, 8, 7)])
def test_generators_golden(port, golden, name, kind, n, d, s):
    g = golden("graphs.npz")
    x = port.generate(kind, n, d, s)
    np.testing.assert_array_equal(x.off, g[name + "_off"])
    np.testing.assert_array_equal(x.tgt, g[name + "_tgt"])


def test_directed_tree_golden(port, golden):
    g = golden("graphs.npz")
    x = port.from_edges(13, [((v - 1) // 3, v) for v in range(1, 13)], undirected=False).ensure_reverse()
    np.testing.assert_array_equal(x.off, g["dtree13_off"])
    np.testing.assert_array_equal(x.rev_off, g["dtree13_roff"])
    np.testing.assert_array_equal(x.rev_tgt, g["dtree13_rtgt"])


@pytest.mark.parametrize("fixture,graph,L", [("expand_small.npz", "pa400", 2),
                                             ("expand_grid.npz", "pa5000", 3)])
def test_expand_golden(port, golden, fixture, graph, L):
    fx = golden(fixture)
    G = csr_from(golden("graphs.npz"), graph)
    for i in range(int(fx["nmb"])):
        p = f"mb{i}"
        e, k, bi = (int(x) for x in fx[p + "_ref"])
        x = port.expand(G, fx[p + "_batch"], fx["fanouts"], int(fx["seed"]), e, k, bi)
        np.testing.assert_array_equal(x.all_vertices, fx[p + "_all"])
        for h in range(L):
            np.testing.assert_array_equal(x.frontier[h], fx[f"{p}_f{h + 1}"])
            np.testing.assert_array_equal(x.indptr[h], fx[f"{p}_ip{h + 1}"])
            np.testing.assert_array_equal(x.edges[h], fx[f"{p}_ed{h + 1}"])


def test_epoch_permutation_golden(port, golden):
    fx = golden("expand_small.npz")
    for e in range(2):
        for k in range(4):
            np.testing.assert_array_equal(
                port.epoch_permutation(fx["roles"], fx["labels"], k, 16, e, 77), fx[f"perm_e{e}_k{k}"])


def test_vip_golden_bitexact(port, golden):
    v = golden("vip.npz")
    gg = golden("graphs.npz")
    hop, tot = port.propagate(csr_from(gg, "path3"), [1, 1], [1.0, 0, 0])
    np.testing.assert_array_equal(hop, v["path3_hop"])
    np.testing.assert_array_equal(tot, v["path3_total"])
    p0 = np.zeros(150)
    p0[5] = 1
    hop, tot = port.propagate(csr_from(gg, "pa150"), [1000] * 3, p0)
    np.testing.assert_array_equal(hop, v["sat_hop"])
    p0 = np.zeros(13)
    p0[0] = 1
    hop, tot = port.propagate(csr_from(gg, "dtree13"), [2, 2], p0)
    np.testing.assert_array_equal(hop, v["dtree_hop"])
    np.testing.assert_array_equal(tot, v["dtree_total"])
    fx = golden("expand_grid.npz")
    G = csr_from(gg, "pa5000")
    for k in range(4):
        p0 = port.initial_probs(fx["roles"], fx["labels"], 4, k, 64)
        np.testing.assert_array_equal(p0, v[f"grid_p0_{k}"])
        hop, tot = port.propagate(G, [15, 10, 5], p0)
        np.testing.assert_array_equal(hop, v[f"grid_hop_{k}"])
        np.testing.assert_array_equal(tot, v[f"grid_total_{k}"])


def test_policy_golden(port, golden):
    pol = golden("policy.npz")
    labels = pol["labels"]
    orders = []
    for k in range(4):
        o, s = port.rank_by_scores(labels, 4, k, pol[f"total_{k}"])
        np.testing.assert_array_equal(o, pol[f"order_{k}"])
        np.testing.assert_array_equal(s, pol[f"score_{k}"])
        orders.append(o)
    o, _ = port.rank_by_scores(np.array([0, 1, 1, 1], np.uint32), 2, 0, np.full(4, 5.0))
    np.testing.assert_array_equal(o, pol["tie_order"])
    oon, ranges = port.build_reorder(labels, 4, np.stack([pol[f"total_{k}"] for k in range(4)]))
    np.testing.assert_array_equal(oon, pol["old_of_new"])
    np.testing.assert_array_equal(ranges, pol["ranges"])


@pytest.mark.parametrize("alpha", [0.0, 0.1, 0.15, 3.0])
def test_cache_and_classify_golden(port, golden, alpha):
    """build_cache bitsets + simulate tallies (commsim.cpp:77-127) recomputed
    from port expansions and port classify."""
    pol = golden("policy.npz")
    labels, roles = pol["labels"], pol["roles"]
    G = csr_from(golden("graphs.npz"), "pa400")
    orders = [pol[f"order_{k}"] for k in range(4)]
    cached, bits = port.build_cache(orders, alpha, 400)
    tag = str(alpha).replace(".", "p")
    np.testing.assert_array_equal(bits, pol[f"bits_{tag}"])
    cells = np.zeros((3, 4, 3), np.uint64)
    for e in range(3):
        for k in range(4):
            for i, b in enumerate(port.epoch_minibatches(roles, labels, k, 16, e, 77)):
                x = port.expand(G, b, [4, 3], 77, e, k, i)
                cells[e, k] += np.array(port.classify(x.all_vertices, labels, k, bits[k]), np.uint64)
    np.testing.assert_array_equal(cells, pol[f"cells_{tag}"])
