"""GPU: the sparse-frontier sampler (vertex-range buckets deduplicated in
shared memory, frontier_sparse.cuh) forced on graphs of every size is
bit-identical to the oracle and to the dense (bitmap) path: frontiers, MFG
row pointers and edges, relabel maps, all_vertices, and the gathered rows
through the bucket-based vertex tiles."""
import ctypes as C

import numpy as np
import pytest

from conftest import csr_from
from test_gpu_sampler import assert_same

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fixture,graph", [("expand_small.npz", "pa400"), ("expand_grid.npz", "pa5000")])
def test_sparse_wave_vs_golden(vk, golden, fixture, graph):
    fx = golden(fixture)
    csr = csr_from(golden("graphs.npz"), graph)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    L = len(fx["fanouts"])
    nmb = int(fx["nmb"])
    s = vk.Sampler(g, fx["fanouts"], int(fx["b"]), nmb, int(fx["seed"]), frontier="sparse")
    batches = [fx[f"mb{i}_batch"] for i in range(nmb)]
    refs = [tuple(int(x) for x in fx[f"mb{i}_ref"]) for i in range(nmb)]
    s.run(batches, refs)
    for i in range(nmb):
        p = f"mb{i}"
        assert_same(s.result(i), L, [fx[f"{p}_f{h + 1}"] for h in range(L)], fx[p + "_all"],
                    [fx[f"{p}_ip{h + 1}"] for h in range(L)], [fx[f"{p}_ed{h + 1}"] for h in range(L)])


@pytest.mark.parametrize("case", range(12))
def test_sparse_random_configs_vs_oracle(vk, port, case):
    """Random configurations (1-3 hops, fanouts 1..40, batches 1..300, waves
    of 1..9) on graphs from one bucket (n <= 2^14) to thousands of buckets,
    with duplicate seeds in some batches; runs twice to check the workspace
    (histograms, look-back status, tickets) resets between runs."""
    rng = np.random.default_rng(5000 + case)
    n = [3000, 16384, 16385, 40000, 200000, 524289, 1000, 100000, 2000000, 65537, 7000, 3000000][case]
    csr = port.generate("pa", n, int(rng.integers(2, 8)), int(rng.integers(0, 99)))
    L = int(rng.integers(1, 4))
    fan = [int(x) for x in rng.choice([1, 2, 3, 5, 8, 10, 15, 17, 25, 33, 40], L)]
    b = int(rng.integers(1, 301))
    nmb = int(rng.integers(1, 10))
    seed = int(rng.integers(0, 1 << 31))
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    s = vk.Sampler(g, fan, b, nmb, seed, frontier="sparse")
    for rep in range(2):
        batches = [rng.integers(0, n, b).astype(np.uint32) for _ in range(nmb)]
        if case % 3:
            batches = [np.unique(x) for x in batches]
        refs = [(int(rng.integers(0, 5)), int(rng.integers(0, 4)), i) for i in range(nmb)]
        s.run(batches, refs)
        for i in range(nmb):
            e, k, bi = refs[i]
            x = port.expand(csr, batches[i], fan, seed, e, k, bi)
            assert_same(s.result(i), L, x.frontier, x.all_vertices, x.indptr, x.edges)


def test_sparse_equals_dense_and_gather(vk, port):
    """Same wave through both representations: identical views; the gather
    over the bucket tiles writes the same rows and tallies as over the dense
    rank words (C3-like community graph, 4 partitions, fp16 rows)."""
    n, K = 400000, 4
    off, tgt, labels = vk.synth_community_powerlaw(n, 12, K, 0.8, 7, 0)
    roles = vk.synth_roles(n, 0.05, 0, 0, 3)
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, 512) for k in range(K)])
    totals = np.stack([x.total for x in vk.propagate(g, [15, 10, 5], p0, with_hops=False)])
    plan = vk.build_cache([vk.rank_by_scores(labels, k, totals[k])[0] for k in range(K)], 0.2, n)
    oon, ranges = vk.build_reorder(labels, K, totals)
    plane = vk.FeaturePlane(n, K, 64, labels, oon, ranges, dtype=1)
    for k in range(K):
        plane.load_partition(k, plan.cached[k], feature_seed=3)
    batches, refs = [], []
    for k in range(K):
        perm = vk.epoch_permutation(roles, labels, k, 512, 0, 42)
        for i in range(3):
            batches.append(perm[i * 512:(i + 1) * 512])
            refs.append((0, k, i))
    outs = {}
    for mode in ("dense", "sparse"):
        s = vk.Sampler(g, [15, 10, 5], 512, len(batches), 42, frontier=mode)
        s.run(batches, refs)
        view = s.view()
        rb = plane.row_bytes
        out, cnt = C.c_void_p(), C.c_void_p()
        vk.check(vk.lib().vk_device_alloc(0, len(batches) * view.all_stride * rb, C.byref(out)))
        vk.check(vk.lib().vk_device_alloc(0, len(batches) * 32, C.byref(cnt)))
        plane.gather(s, out.value, view.all_stride, cnt.value)
        counts = np.zeros(len(batches) * 4, np.uint64)
        vk.check(vk.lib().vk_memcpy(counts.ctypes.data, cnt, counts.nbytes, 2))
        res = [s.result(i) for i in range(len(batches))]
        rows = []
        for i, r in enumerate(res):
            buf = np.zeros(len(r.all_vertices) * rb, np.uint8)
            vk.check(vk.lib().vk_memcpy(buf.ctypes.data, out.value + i * view.all_stride * rb, buf.nbytes, 2))
            rows.append(buf)
        vk.lib().vk_device_free(out)
        vk.lib().vk_device_free(cnt)
        outs[mode] = (res, rows, counts)
    (rd, rowd, cd), (rs, rows_, cs) = outs["dense"], outs["sparse"]
    np.testing.assert_array_equal(cd, cs)
    for i in range(len(batches)):
        a, b_ = rd[i], rs[i]
        np.testing.assert_array_equal(a.all_vertices, b_.all_vertices)
        for h in range(3):
            np.testing.assert_array_equal(a.frontier[h], b_.frontier[h])
            np.testing.assert_array_equal(a.mfg_indptr[h], b_.mfg_indptr[h])
            np.testing.assert_array_equal(a.mfg_dst[h], b_.mfg_dst[h])
        for h in range(4):
            np.testing.assert_array_equal(a.all_index[h], b_.all_index[h])
        np.testing.assert_array_equal(rowd[i], rows_[i])
        exp = port.features(3, 64, a.all_vertices, fp16=True)
        np.testing.assert_array_equal(rows_[i].view(np.uint16), exp.view(np.uint16).ravel())


@pytest.mark.parametrize("frontier", ["sparse", "dense"])
def test_isolated_seeds_empty_frontiers(vk, port, frontier):
    """Seeds without neighbours (empty F_1 and every later hop for that
    minibatch), hubs beside them, and a graph spanning several buckets: both
    representations equal the oracle, including the empty levels."""
    from oracle.oracle import CSR
    n = 600000
    rng = np.random.default_rng(11)
    # vertices >= 300000 are isolated; the rest form a sparse random graph
    # with a few hubs
    src = rng.integers(0, 300000, 900000).astype(np.uint32)
    dst = rng.integers(0, 300000, 900000).astype(np.uint32)
    hubs = rng.integers(0, 300000, 5).astype(np.uint32)
    src = np.concatenate([src, np.repeat(hubs, 4000)])
    dst = np.concatenate([dst, rng.integers(0, 300000, 20000).astype(np.uint32)])
    keep = src != dst
    u = np.concatenate([src[keep], dst[keep]])
    v = np.concatenate([dst[keep], src[keep]])
    key = np.unique(u.astype(np.uint64) << 32 | v)
    u, v = (key >> 32).astype(np.uint32), (key & 0xffffffff).astype(np.uint32)
    off = np.zeros(n + 1, np.uint64)
    np.add.at(off, u.astype(np.int64) + 1, 1)
    off = np.cumsum(off).astype(np.uint64)
    csr = CSR(n, off, v)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    fan = [10, 5, 3]
    batches = [np.arange(300000, 300100, dtype=np.uint32),          # isolated only
               np.concatenate([hubs, np.arange(300000, 300050, dtype=np.uint32)]),
               rng.integers(0, 300000, 200).astype(np.uint32),
               np.array([599999], np.uint32)]                         # last vertex, isolated
    refs = [(0, 0, i) for i in range(len(batches))]
    s = vk.Sampler(g, fan, 200, len(batches), 77, frontier=frontier)
    s.run(batches, refs)
    for i, bt in enumerate(batches):
        x = port.expand(csr, bt, fan, 77, 0, 0, i)
        assert_same(s.result(i), 3, x.frontier, x.all_vertices, x.indptr, x.edges)
    assert len(port.expand(csr, batches[0], fan, 77, 0, 0, 0).frontier[0]) == 0
