"""GPU, full size: BASELINE configs[2] (C3, ogbn-products-shaped, 2.45 M
vertices / 122 M CSR slots) in the bench's own wave of 128 minibatches, and a
sparse 8 M-vertex graph whose frontiers take the wide-tile compaction path.

Sampled minibatches of each wave are checked bit-exact against the oracle
(frontiers, all_vertices, MFG row pointers and edges, relabel maps, gathered
rows, local/cache/miss tallies); every minibatch of the wave is checked for the
size-independent invariants of SURVEY §8a (sorted distinct frontiers whose
union with the batch is all_vertices, MFG row lengths min(f, deg), sampled
edges are CSR neighbours, relabel maps round-trip)."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import CSR

pytestmark = pytest.mark.gpu


def assert_invariants(r, off, tgt, fan, rng):
    a = r.all_vertices
    assert np.all(np.diff(a.astype(np.int64)) > 0)
    parts = [r.batch]
    for h, f in enumerate(fan):
        fr = r.frontier[h]
        assert np.all(np.diff(fr.astype(np.int64)) > 0)
        parts.append(fr)
        src = r.batch if h == 0 else r.frontier[h - 1]
        deg = (off[src.astype(np.int64) + 1] - off[src]).astype(np.int64)
        ip = r.mfg_indptr[h].astype(np.int64)
        np.testing.assert_array_equal(np.diff(ip), np.minimum(f, deg))
        dst = r.mfg_dst[h]
        assert dst.size == ip[-1] and (dst.size == 0 or dst.max() < fr.size)
        # a sample of edges: the drawn id is a CSR neighbour of its source
        if dst.size:
            e = rng.integers(0, dst.size, min(2000, dst.size))
            s = np.searchsorted(ip, e, side="right") - 1
            v, u = src[s].astype(np.int64), fr[dst[e]]
            for vi, ui in zip(v[:200], u[:200]):
                assert ui in tgt[off[vi]:off[vi + 1]]
    np.testing.assert_array_equal(np.unique(np.concatenate(parts)), a)
    np.testing.assert_array_equal(a[r.all_index[0]], r.batch)
    for h in range(len(fan)):
        np.testing.assert_array_equal(a[r.all_index[h + 1]], r.frontier[h])


def assert_bit_exact(r, x, L):
    np.testing.assert_array_equal(r.all_vertices, x.all_vertices)
    for h in range(L):
        np.testing.assert_array_equal(r.frontier[h], x.frontier[h])
        np.testing.assert_array_equal(r.mfg_indptr[h], x.indptr[h])
        np.testing.assert_array_equal(r.frontier[h][r.mfg_dst[h]], x.edges[h])


@pytest.fixture(scope="module")
def c3(vk):
    n = 2_449_029
    off, tgt, labels = vk.synth_community_powerlaw(n, 25, 8, 0.8, 7, 0)
    roles = vk.synth_roles(n, 0.08, 0, 0, 3)
    return n, off, tgt, labels, roles


def test_c3_wave_sample_and_gather(vk, port, c3):
    n, off, tgt, labels, roles = c3
    K, b, fan, dim, seed, fseed, M = 8, 1024, [15, 10, 5], 100, 42, 1234, 128
    csr = CSR(n, off, tgt)
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    # cache plan / store layout from arbitrary (seeded) scores: the gather
    # must be exact for any VIP ordering
    scores = np.random.default_rng(5).random((K, n))
    orders = [vk.rank_by_scores(labels, k, scores[k])[0] for k in range(K)]
    plan = vk.build_cache(orders, 0.2, n)
    oon, ranges = vk.build_reorder(labels, K, scores)
    plane = vk.FeaturePlane(n, K, dim, labels, oon, ranges)
    for k in range(K):
        plane.load_partition(k, plan.cached[k], feature_seed=fseed)
    batches, refs = [], []
    for k in range(K):
        perm = vk.epoch_permutation(roles, labels, k, b, 0, seed)
        for i in range(M // K):
            batches.append(perm[i * b:(i + 1) * b])
            refs.append((0, k, i))
    s = vk.Sampler(g, fan, b, M, seed)
    s.run(batches, refs)
    view = s.view()
    rb = plane.row_bytes
    out, cnt = C.c_void_p(), C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(0, M * view.all_stride * rb, C.byref(out)))
    vk.check(vk.lib().vk_device_alloc(0, M * 32, C.byref(cnt)))
    try:
        plane.gather(s, out.value, view.all_stride, cnt.value)
        counts = np.zeros(M * 4, np.uint64)
        vk.check(vk.lib().vk_memcpy(counts.ctypes.data, cnt, counts.nbytes, 2))
        counts = counts.reshape(M, 4)
        rng = np.random.default_rng(0)
        for i in range(M):
            r = s.result(i)
            assert_invariants(r, off, tgt, fan, rng)
            e, k, bi = refs[i]
            loc, hit, miss = port.classify(r.all_vertices, labels, k, plan.member_bits[k])
            assert tuple(int(c) for c in counts[i][:3]) == (loc, hit, miss)
            if i % 37 == 0 or i == M - 1:  # bit-exact sample of the wave
                x = port.expand(csr, batches[i], fan, seed, e, k, bi)
                assert_bit_exact(r, x, len(fan))
                rows = np.zeros((len(r.all_vertices), dim), np.float32)
                vk.check(vk.lib().vk_memcpy(rows.ctypes.data, out.value + i * view.all_stride * rb,
                                            rows.nbytes, 2))
                exp = port.features(fseed, dim, r.all_vertices)
                np.testing.assert_array_equal(rows.view(np.uint32), exp.view(np.uint32))
    finally:
        vk.lib().vk_device_free(out)
        vk.lib().vk_device_free(cnt)


def test_sparse_graph_wide_tile_compaction(vk, port):
    """8 M vertices, batch 64: every hop's expected density is far below one
    id per 64-bit word. The dense (bitmap) representation, forced here, takes
    its wide-tile compaction (16 words per thread, nonzero-word) path; the
    automatic choice for this shape is the sparse (bucket) one, and both are
    bit-exact against the oracle and identical to each other."""
    n = 8_000_000
    off, tgt, labels = vk.synth_community_powerlaw(n, 3, 4, 0.8, 11, 0)
    roles = vk.synth_roles(n, 0.01, 0, 0, 5)
    csr = CSR(n, off, tgt)
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    fan, b, M, seed = [15, 10, 5], 64, 96, 17
    batches, refs = [], []
    for k in range(4):
        perm = vk.epoch_permutation(roles, labels, k, b, 2, seed)
        for i in range(M // 4):
            batches.append(perm[i * b:(i + 1) * b])
            refs.append((2, k, i))
    s = vk.Sampler(g, fan, b, M, seed, frontier="dense")
    auto = vk.Sampler(g, fan, b, M, seed)
    for rep in range(2):  # the second run checks the workspace was left clean
        s.run(batches, refs)
        auto.run(batches, refs)
        rng = np.random.default_rng(rep)
        for i in range(M):
            r = s.result(i)
            assert_invariants(r, off, tgt, fan, rng)
            q = auto.result(i)
            np.testing.assert_array_equal(q.all_vertices, r.all_vertices)
            for h in range(len(fan)):
                np.testing.assert_array_equal(q.mfg_dst[h], r.mfg_dst[h])
                np.testing.assert_array_equal(q.all_index[h + 1], r.all_index[h + 1])
            if i % 23 == 0:
                e, k, bi = refs[i]
                assert_bit_exact(r, port.expand(csr, batches[i], fan, seed, e, k, bi), len(fan))
