"""GPU: the batched sampler (K5/K6 + MFG + relabel) vs the oracle. Bit-exact:
frontiers, all_vertices, MFG row pointers, MFG edges (global id = F_h[dst]) and
the relabel maps."""
import numpy as np
import pytest

from conftest import csr_from

pytestmark = pytest.mark.gpu


def dev_graph(vk, csr):
    return vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)


def assert_same(gpu, L, frontiers, all_vertices, indptr=None, edges=None):
    np.testing.assert_array_equal(gpu.all_vertices, all_vertices)
    for h in range(L):
        np.testing.assert_array_equal(gpu.frontier[h], frontiers[h])
        if indptr is not None:
            np.testing.assert_array_equal(gpu.mfg_indptr[h], indptr[h])
            np.testing.assert_array_equal(gpu.frontier[h][gpu.mfg_dst[h]], edges[h])
    # relabel maps: all_vertices[all_index[h]] == F_h (h = 0 is the batch)
    np.testing.assert_array_equal(gpu.all_vertices[gpu.all_index[0]], gpu.batch)
    for h in range(L):
        np.testing.assert_array_equal(gpu.all_vertices[gpu.all_index[h + 1]], gpu.frontier[h])


@pytest.mark.parametrize("fixture,graph", [("expand_small.npz", "pa400"), ("expand_grid.npz", "pa5000")])
def test_wave_vs_golden(vk, golden, fixture, graph):
    fx = golden(fixture)
    csr = csr_from(golden("graphs.npz"), graph)
    g = dev_graph(vk, csr)
    L = len(fx["fanouts"])
    nmb = int(fx["nmb"])
    s = vk.Sampler(g, fx["fanouts"], int(fx["b"]), nmb, int(fx["seed"]))
    batches = [fx[f"mb{i}_batch"] for i in range(nmb)]
    refs = [tuple(int(x) for x in fx[f"mb{i}_ref"]) for i in range(nmb)]
    s.run(batches, refs)
    for i in range(nmb):
        p = f"mb{i}"
        r = s.result(i)
        np.testing.assert_array_equal(r.batch, batches[i])
        assert_same(r, L, [fx[f"{p}_f{h + 1}"] for h in range(L)], fx[p + "_all"],
                    [fx[f"{p}_ip{h + 1}"] for h in range(L)], [fx[f"{p}_ed{h + 1}"] for h in range(L)])


def test_c1_epoch_slice_vs_oracle(vk, port):
    """C1 (BASELINE configs[0]): PA 1e5/d=10, roles 0.1, K=1, b=1024,
    (15,10,5), SeedSpec{42}: the first 8 minibatches of epoch 0 in one wave."""
    csr = port.generate("pa", 100000, 10, 7)
    roles = port.make_roles(csr.n, 0.1, 0, 0, 3)
    labels = np.zeros(csr.n, np.uint32)
    perm = port.epoch_permutation(roles, labels, 0, 1024, 0, 42)
    np.testing.assert_array_equal(perm, vk.epoch_permutation(roles, labels, 0, 1024, 0, 42))
    batches = [perm[i * 1024:(i + 1) * 1024] for i in range(8)]
    g = dev_graph(vk, csr)
    s = vk.Sampler(g, [15, 10, 5], 1024, 8, 42)
    s.run(batches, [(0, 0, i) for i in range(8)])
    for i in range(8):
        x = port.expand(csr, batches[i], [15, 10, 5], 42, 0, 0, i)
        assert_same(s.result(i), 3, x.frontier, x.all_vertices, x.indptr, x.edges)


def test_ragged_last_batch_and_reuse(vk, port):
    csr = port.generate("pa", 30000, 5, 11)
    roles = port.make_roles(csr.n, 0.2, 0, 0, 2)
    labels = (np.arange(csr.n) % 3).astype(np.uint32)
    g = dev_graph(vk, csr)
    s = vk.Sampler(g, [10, 5], 300, 6, 9)
    for e in range(2):  # the second run reuses (and must fully reset) the workspace
        perm = port.epoch_permutation(roles, labels, 1, 300, e, 9)
        nb = (len(perm) + 299) // 300
        assert nb >= 6
        idx = list(range(nb - 6, nb))  # ends with the ragged batch
        batches = [perm[i * 300:(i + 1) * 300] for i in idx]
        assert len(batches[-1]) < 300
        s.run(batches, [(e, 1, i) for i in idx])
        for j, i in enumerate(idx):
            x = port.expand(csr, batches[j], [10, 5], 9, e, 1, i)
            assert_same(s.result(j), 2, x.frontier, x.all_vertices, x.indptr, x.edges)


def test_large_fanout_path(vk, port):
    """fanout > 32 with hub vertices of higher degree (128-entry FY state)."""
    csr = port.generate("pa", 20000, 8, 4)
    batch = np.argsort(-np.diff(csr.off).astype(np.int64))[:64].astype(np.uint32)  # hubs
    g = dev_graph(vk, csr)
    s = vk.Sampler(g, [40, 3], 64, 1, 5)
    s.run([batch], [(1, 0, 2)])
    x = port.expand(csr, batch, [40, 3], 5, 1, 0, 2)
    assert_same(s.result(0), 2, x.frontier, x.all_vertices, x.indptr, x.edges)


def test_saturating_and_duplicates(vk, port, golden):
    csr = csr_from(golden("graphs.npz"), "pa120")
    g = dev_graph(vk, csr)
    x = vk.expand(g, [3, 17, 3], [1000, 1000], 1, (0, 0, 0))  # duplicate seed
    y = port.expand(csr, [3, 17, 3], [1000, 1000], 1, 0, 0, 0)
    assert_same(x, 2, y.frontier, y.all_vertices, y.indptr, y.edges)


def test_expand_single_and_errors(vk, port, golden):
    csr = csr_from(golden("graphs.npz"), "uni200")
    g = dev_graph(vk, csr)
    x = vk.expand(g, [1, 2, 3, 50, 51], [3, 2, 2], 5, (7, 0, 3))
    y = port.expand(csr, [1, 2, 3, 50, 51], [3, 2, 2], 5, 7, 0, 3)
    assert_same(x, 3, y.frontier, y.all_vertices, y.indptr, y.edges)
    with pytest.raises(vk.SamplingError):
        vk.expand(g, [], [3, 2], 5)
    with pytest.raises(vk.ParameterError):
        vk.expand(g, [1], [3, 0], 5)
    s = vk.Sampler(g, [3, 2], 8, 2, 5)
    with pytest.raises(vk.RangeError):
        s.run([[1, 999]], [(0, 0, 0)])
    with pytest.raises(vk.SamplingError):
        s.run([[1], []], [(0, 0, 0), (0, 0, 1)])


def test_device_rng_matches_reference_draws(vk, golden, port):
    """RngStream on the device (FP64-reciprocal modulo) == reference draws,
    including bound 1, powers of two, 2^32, >= 2^40 (slow path) and 2^63."""
    g = golden("rng.npz")
    for i, b in enumerate(g["bounds"]):
        np.testing.assert_array_equal(vk.stream_draws(12345 + i, int(b), 64), g["draws"][i])
    rng = np.random.default_rng(0)
    for b in list(rng.integers(2, 1 << 32, 200)) + [(1 << 40) - 1, 3, 7, 1 << 31, (1 << 32) - 5]:
        key = int(rng.integers(0, 1 << 62))
        np.testing.assert_array_equal(vk.stream_draws(key, int(b), 300), port.stream_draws(key, int(b), 300))


def test_seed_keys_replay_vs_reference(vk, ref, golden):
    """seed_keys replay (sampling.hpp:46-64): on a relabelled graph with
    seed_keys = old_of_new the device expansion is bit-exact with the
    reference's keyed expand, and maps back onto the original graph's
    expansion vertex for vertex."""
    from oracle.oracle import CSR
    csr = csr_from(golden("graphs.npz"), "pa5000")
    n = csr.n
    rng = np.random.default_rng(3)
    K = 4
    labels = rng.integers(0, K, n).astype(np.uint32)
    roles = np.zeros(n, np.uint8)
    oon, _ = vk.build_reorder(labels, K, rng.random((K, n)))
    g = dev_graph(vk, csr)
    ng, r2, l2 = vk.apply_reorder(g, roles, labels, oon)
    noff, ntgt = ng.forward()
    ncsr = CSR(n, noff, ntgt)
    new_of_old = np.empty(n, np.uint32)
    new_of_old[oon] = np.arange(n, dtype=np.uint32)
    fan = [15, 10, 5]
    for i in range(3):
        batch_old = rng.choice(n, 64, replace=False).astype(np.uint32)
        batch_new = new_of_old[batch_old]
        got = vk.expand(ng, batch_new, fan, 42, (1, 2, i), seed_keys=oon)
        exp = ref.expand(ncsr, batch_new, fan, 42, 1, 2, i, seed_keys=oon)
        assert_same(got, 3, exp.frontier, exp.all_vertices, exp.indptr, exp.edges)
        orig = vk.expand(g, batch_old, fan, 42, (1, 2, i))
        np.testing.assert_array_equal(np.sort(oon[got.all_vertices]), orig.all_vertices)
        for h in range(3):
            np.testing.assert_array_equal(np.sort(oon[got.frontier[h]]), orig.frontier[h])
    # replay off again: plain expansion of the relabelled graph
    plain = vk.expand(ng, batch_new, fan, 42, (1, 2, 2))
    x = ref.expand(ncsr, batch_new, fan, 42, 1, 2, 2)
    assert_same(plain, 3, x.frontier, x.all_vertices, x.indptr, x.edges)


@pytest.mark.parametrize("case", range(16))
def test_random_configs_vs_oracle(vk, port, case):
    """Seeded random sampler configurations around the code-path boundaries:
    1-3 hops, fanouts 1..40 (register / shared / local Fisher-Yates), batch
    sizes 1..300, waves of 1..9, graphs on both sides of the small-graph
    (shared-memory compaction) limit of 524,288 vertices."""
    rng = np.random.default_rng(1000 + case)
    n = [3000, 40000, 524288, 524289, 200000, 7000, 524288, 600000,
         1000, 65536, 65537, 300000, 524224, 12345, 100000, 2000000][case]
    d = int(rng.integers(2, 8))
    csr = port.generate("pa", n, d, int(rng.integers(0, 99)))
    L = int(rng.integers(1, 4))
    fan = [int(x) for x in rng.choice([1, 2, 3, 5, 8, 10, 15, 17, 25, 33, 40], L)]
    b = int(rng.integers(1, 301))
    nmb = int(rng.integers(1, 10))
    seed = int(rng.integers(0, 1 << 31))
    g = dev_graph(vk, csr)
    batches = [np.unique(rng.integers(0, n, b)).astype(np.uint32) for _ in range(nmb)]
    rng.shuffle(batches[0])  # batch order is expand's hop-1 visiting order
    refs = [(int(rng.integers(0, 5)), int(rng.integers(0, 4)), i) for i in range(nmb)]
    s = vk.Sampler(g, fan, b, nmb, seed)
    s.run(batches, refs)
    for i in range(nmb):
        e, k, bi = refs[i]
        x = port.expand(csr, batches[i], fan, seed, e, k, bi)
        assert_same(s.result(i), L, x.frontier, x.all_vertices, x.indptr, x.edges)
