"""GPU: vipkit::simulate / the alpha axis of sweep through
vk_simulate vs the reference's own tallies: the golden CommReport cells of the
reference's SmallSetup (written by the real reference, oracle/make_golden.py)
and, at C2 size, the live compiled reference (oracle/_ref). Exact counts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_small_setup_cells_vs_golden(vk, port, golden):
    pol = golden("policy.npz")
    csr = port.generate("pa", 400, 4, 15)
    roles = port.make_roles(400, 0.25, 0, 0, 6)
    np.testing.assert_array_equal(roles, pol["roles"])
    labels = pol["labels"]
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    orders = [pol[f"order_{k}"] for k in range(4)]
    alphas = (0.0, 0.1, 0.15, 3.0)
    plans = [vk.build_cache(orders, a, 400) for a in alphas]
    for a, plan in zip(alphas, plans):
        np.testing.assert_array_equal(plan.member_bits, pol["bits_" + str(a).replace(".", "p")])
    # one plan at a time (CachePlan semantics) ...
    for a, plan in zip(alphas, plans):
        cells = vk.simulate(g, roles, labels, 4, [4, 3], 16, 3, 77, plan.cached)
        np.testing.assert_array_equal(cells, pol["cells_" + str(a).replace(".", "p")])
    # ... and all four from one expansion pass (nested ranking prefixes)
    takes = [[len(p.cached[k]) for k in range(4)] for p in plans]
    multi = vk.simulate(g, roles, labels, 4, [4, 3], 16, 3, 77, plans[-1].cached, takes=takes, wave=5)
    for i, a in enumerate(alphas):
        np.testing.assert_array_equal(multi[i], pol["cells_" + str(a).replace(".", "p")])


def test_c2_alpha_sweep_vs_reference(vk, port, ref):
    """C2-shaped (169,343 vertices, PA d=7, 2 partitions): one epoch, VIP
    rankings, alpha in {0, 0.1, 0.2} against the reference's simulate."""
    n, K, b, fan, seed = 169_343, 2, 1024, [15, 10, 5], 42
    csr = port.generate("pa", n, 7, 7)
    roles = port.make_roles(n, 0.537, 0, 0, 3)
    labels = ((np.arange(n, dtype=np.uint64) * 2654435761) % K).astype(np.uint32)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, b) for k in range(K)])
    totals = np.stack([s.total for s in vk.propagate(g, fan, p0, with_hops=False)])
    orders = [vk.rank_by_scores(labels, k, totals[k])[0] for k in range(K)]
    alphas = (0.0, 0.1, 0.2)
    plans = [vk.build_cache(orders, a, n) for a in alphas]
    takes = [[len(p.cached[k]) for k in range(K)] for p in plans]
    got = vk.simulate(g, roles, labels, K, fan, b, 1, seed, plans[-1].cached, takes=takes)
    for i, plan in enumerate(plans):
        exp = ref.simulate(csr, roles, labels, K, fan, b, 1, seed, plan.cached)
        np.testing.assert_array_equal(got[i], exp)
    misses = [int(got[i][..., 2].sum()) for i in range(len(alphas))]
    assert misses[0] > misses[1] > misses[2]  # the VIP cache cuts remote misses


def test_simulate_errors(vk, port):
    csr = port.generate("pa", 300, 3, 1)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    roles = port.make_roles(300, 0.3, 0, 0, 2)
    labels = np.zeros(300, np.uint32)
    labels[:5] = 1
    roles_no_train_in_1 = roles.copy()
    roles_no_train_in_1[:5] = 1
    empty = [np.zeros(0, np.uint32)] * 2
    with pytest.raises(vk.SamplingError):
        vk.simulate(g, roles_no_train_in_1, labels, 2, [3], 8, 1, 1, empty)
    with pytest.raises(vk.ParameterError):
        vk.simulate(g, roles, labels, 2, [3], 0, 1, 1, empty)
    with pytest.raises(vk.FormatError):
        vk.simulate(g, roles, labels, 1, [3], 8, 1, 1, empty[:1])


@pytest.mark.parametrize("K,k,b,fan,S", [(1, 0, 64, [10, 5], 3), (4, 2, 32, [15, 10, 5], 2)])
def test_empirical_vip_vs_reference(vk, port, ref, K, k, b, fan, S):
    """vipkit::empirical_vip (vip.cpp:85-105): frequencies bit-identical to
    the live reference (same derived streams, same double division)."""
    csr = port.generate("pa", 20000, 6, 13)
    roles = port.make_roles(csr.n, 0.1, 0, 0, 4)
    labels = (np.arange(csr.n) % K).astype(np.uint32)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    got = vk.empirical_vip(g, roles, labels, K, k, b, fan, S, 42)
    exp = ref.empirical_vip(csr, roles, labels, K, k, b, fan, S, 42)
    np.testing.assert_array_equal(got, exp)
    assert got.max() == 1.0 and 0.0 < got.mean() < 1.0


def test_simulate_with_seed_keys_is_reorder_invariant(vk, port, ref):
    """test_reorder.cpp:154-179 + SimulateOptions::seed_keys: after
    apply_reorder, simulate with seed_keys = old_of_new reproduces the
    original graph's local/miss cells; bit-exact vs the keyed reference."""
    from oracle.oracle import CSR
    csr = port.generate("pa", 2500, 4, 51)
    n, K = csr.n, 2
    roles = port.make_roles(n, 0.3, 0, 0, 2)
    labels = (np.arange(n) % K).astype(np.uint32)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, 8) for k in range(K)])
    totals = np.stack([s.total for s in vk.propagate(g, [3, 2], p0, with_hops=False)])
    oon, _ = vk.build_reorder(labels, K, totals)
    ng, r2, l2 = vk.apply_reorder(g, roles, labels, oon)
    noff, ntgt = ng.forward()
    empty = [np.zeros(0, np.uint32)] * K
    before = vk.simulate(g, roles, labels, K, [3, 2], 8, 3, 2024, empty)
    after = vk.simulate(ng, r2, l2, K, [3, 2], 8, 3, 2024, empty, seed_keys=oon)
    np.testing.assert_array_equal(before[..., 0], after[..., 0])
    np.testing.assert_array_equal(before[..., 2], after[..., 2])
    exp = ref.simulate(CSR(n, noff, ntgt), r2, l2, K, [3, 2], 8, 3, 2024, empty, seed_keys=oon)
    np.testing.assert_array_equal(after, exp)


def test_access_counts_vs_reference_expansions(vk, port, ref, golden):
    """The oracle policy's access counts (commsim.cpp:155-166) equal a
    histogram of the reference's own expansions in for_each_expansion order."""
    pol = golden("policy.npz")
    csr = port.generate("pa", 400, 4, 15)
    roles, labels = pol["roles"], pol["labels"]
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    got = vk.access_counts(g, roles, labels, 4, [4, 3], 16, 3, 77)
    exp = np.zeros((4, 400))
    for e in range(3):
        for k in range(4):
            perm = ref.epoch_permutation(roles, labels, k, 16, e, 77, K=4)
            for i in range((len(perm) + 15) // 16):
                x = ref.expand(csr, perm[i * 16:(i + 1) * 16], [4, 3], 77, e, k, i, with_mfg=False)
                exp[k, x.all_vertices] += 1
    np.testing.assert_array_equal(got, exp)
