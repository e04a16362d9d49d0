"""GPU: ranking, reorder, cache membership and the classify+gather kernel vs
the oracle. Bit-exact rows (fp32 and fp16) and exact local/cache/miss tallies."""
import ctypes as C

import numpy as np
import pytest

from conftest import csr_from

pytestmark = pytest.mark.gpu


def test_rank_by_scores_bit_exact(vk, port, golden):
    pol = golden("policy.npz")
    for k in range(4):
        o, s = vk.rank_by_scores(pol["labels"], k, pol[f"total_{k}"])
        np.testing.assert_array_equal(o, pol[f"order_{k}"])
        np.testing.assert_array_equal(s, pol[f"score_{k}"])
    o, _ = vk.rank_by_scores(np.array([0, 1, 1, 1], np.uint32), 0, np.full(4, 5.0))
    np.testing.assert_array_equal(o, pol["tie_order"])
    rng = np.random.default_rng(3)
    n = 200000
    labels = rng.integers(0, 5, n).astype(np.uint32)
    scores = np.round(rng.random(n), 3)           # many ties
    scores[rng.integers(0, n, 5000)] = 0.0
    scores[rng.integers(0, n, 5000)] = -0.0        # -0.0 ties +0.0 (policies.cpp:28)
    scores[rng.integers(0, n, 100)] = 1.0
    for k in (0, 4):
        o1, s1 = vk.rank_by_scores(labels, k, scores)
        o2, s2 = port.rank_by_scores(labels, 5, k, scores)
        np.testing.assert_array_equal(o1, o2)
    with pytest.raises(vk.ShapeError):
        vk.rank_by_scores(labels, 0, scores[:-1])


def test_build_reorder_bit_exact(vk, golden):
    pol = golden("policy.npz")
    oon, ranges = vk.build_reorder(pol["labels"], 4, np.stack([pol[f"total_{k}"] for k in range(4)]))
    np.testing.assert_array_equal(oon, pol["old_of_new"])
    np.testing.assert_array_equal(ranges, pol["ranges"])


def _pipeline(vk, port, csr, roles, labels, K, fan, b, alpha, seed, dim, dtype, feature_seed, nmb):
    """VIP -> rank -> cache -> reorder -> plane(all K resident) -> sample -> gather."""
    n = csr.n
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, b) for k in range(K)])
    scores = vk.propagate(g, fan, p0, with_hops=False)
    totals = np.stack([s.total for s in scores])
    orders = [vk.rank_by_scores(labels, k, totals[k])[0] for k in range(K)]
    plan = vk.build_cache(orders, alpha, n)
    oon, ranges = vk.build_reorder(labels, K, totals)
    plane = vk.FeaturePlane(n, K, dim, labels, oon, ranges, dtype=dtype)
    for k in range(K):
        plane.load_partition(k, plan.cached[k], feature_seed=feature_seed)
    batches, refs = [], []
    for k in range(K):
        perm = vk.epoch_permutation(roles, labels, k, b, 0, seed)
        for i in range(min(nmb, (len(perm) + b - 1) // b)):
            batches.append(perm[i * b:(i + 1) * b])
            refs.append((0, k, i))
    s = vk.Sampler(g, fan, b, len(batches), seed)
    s.run(batches, refs)
    view = s.view()
    rb = plane.row_bytes
    out_ptr = C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(0, len(batches) * view.all_stride * rb, C.byref(out_ptr)))
    cnt_ptr = C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(0, len(batches) * 32, C.byref(cnt_ptr)))
    plane.gather(s, out_ptr.value, view.all_stride, cnt_ptr.value)
    counts = np.zeros(len(batches) * 4, np.uint64)
    vk.check(vk.lib().vk_memcpy(counts.ctypes.data, cnt_ptr, counts.nbytes, 2))
    counts = counts.reshape(-1, 4)
    _, _, al = s.sizes()
    rows = []
    for i in range(len(batches)):
        buf = np.zeros(int(al[i]) * rb, np.uint8)
        vk.check(vk.lib().vk_memcpy(buf.ctypes.data, out_ptr.value + i * view.all_stride * rb, buf.nbytes, 2))
        rows.append(buf)
    vk.lib().vk_device_free(out_ptr)
    vk.lib().vk_device_free(cnt_ptr)
    return dict(plan=plan, plane=plane, sampler=s, batches=batches, refs=refs, counts=counts,
                rows=rows, totals=totals, g=g)


@pytest.mark.parametrize("dtype,dim", [(0, 64), (1, 128), (0, 100), (0, 3)])
def test_gather_rows_and_tallies(vk, port, golden, dtype, dim):
    fx = golden("expand_grid.npz")
    csr = csr_from(golden("graphs.npz"), "pa5000")
    roles, labels = fx["roles"], fx["labels"]
    r = _pipeline(vk, port, csr, roles, labels, 4, [15, 10, 5], 64, 0.2, 42, dim, dtype, 1234, 3)
    plan = r["plan"]
    for i, (e, k, bi) in enumerate(r["refs"]):
        x = port.expand(csr, r["batches"][i], [15, 10, 5], 42, e, k, bi)
        exp = port.features(1234, dim, x.all_vertices, fp16=dtype == 1)
        got = r["rows"][i].view(np.float16 if dtype == 1 else np.float32).reshape(-1, dim)
        np.testing.assert_array_equal(got.view(np.uint16 if dtype == 1 else np.uint32),
                                      exp.view(np.uint16 if dtype == 1 else np.uint32))
        loc, hit, miss = port.classify(x.all_vertices, labels, k, plan.member_bits[k])
        assert tuple(int(c) for c in r["counts"][i][:3]) == (loc, hit, miss)
        assert r["counts"][i][3] == 0  # single GPU: no miss crosses NVLink
    # cache membership == CachePlan::is_cached
    for k in range(4):
        for v in list(plan.cached[k][:20]) + [0, 1, 2, 3]:
            assert r["plane"].is_cached(k, int(v)) == plan.is_cached(k, int(v))


def test_cache_reduces_misses(vk, port):
    """Miss rows fall as alpha grows (nested prefix caches), alpha = 0 has no hits."""
    csr = port.generate("pa", 20000, 6, 9)
    roles = port.make_roles(csr.n, 0.1, 0, 0, 3)
    labels = (np.arange(csr.n) % 4).astype(np.uint32)
    prev = None
    for alpha in (0.0, 0.1, 0.3, 3.0):
        r = _pipeline(vk, port, csr, roles, labels, 4, [10, 5], 128, alpha, 7, 16, 0, 5, 2)
        miss = int(r["counts"][:, 2].sum())
        hits = int(r["counts"][:, 1].sum())
        if alpha == 0.0:
            assert hits == 0
        if alpha == 3.0:
            assert miss == 0
        if prev is not None:
            assert miss <= prev
        prev = miss


@pytest.mark.parametrize("graph,directed", [("pa5000", False), ("dtree13", True)])
def test_apply_reorder_vs_reference(vk, ref, golden, graph, directed):
    """apply_reorder (reorder.cpp:36-70) on the device: relabelled forward
    and reverse CSR, roles and labels bit-exact vs the live reference."""
    csr = csr_from(golden("graphs.npz"), graph)
    n = csr.n
    rng = np.random.default_rng(7)
    K = 3
    labels = rng.integers(0, K, n).astype(np.uint32)
    roles = rng.integers(0, 3, n).astype(np.uint8)
    scores = rng.random((K, n))
    oon, _ = vk.build_reorder(labels, K, scores)
    if directed:
        g = vk.Graph.from_csr(csr.off, csr.tgt, validate=True)
    else:
        g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    ng, r2, l2 = vk.apply_reorder(g, roles, labels, oon)
    exp, er, el = ref.apply_reorder(csr, roles, labels, K, oon)
    off, tgt = ng.forward()
    roff, rtgt = ng.reverse()
    np.testing.assert_array_equal(off, exp.off)
    np.testing.assert_array_equal(tgt, exp.tgt)
    np.testing.assert_array_equal(roff, exp.rev_off)
    np.testing.assert_array_equal(rtgt, exp.rev_tgt)
    np.testing.assert_array_equal(r2, er)
    np.testing.assert_array_equal(l2, el)
    bad = oon.copy()
    bad[0] = bad[1]
    with pytest.raises(vk.ShapeError):
        vk.apply_reorder(g, roles, labels, bad)
    with pytest.raises(vk.ShapeError):
        vk.apply_reorder(g, roles, labels, oon[:-1])


def test_apply_reorder_c3_scale(vk, port):
    """BASELINE C3 shape (2.45 M vertices, 122 M slots): the relabelled graph
    is isomorphic (degree multiset, sorted rows, every edge maps back) and a
    sampled minibatch of the relabelled graph expands bit-exact vs the oracle."""
    from oracle.oracle import CSR
    n = 2_449_029
    off, tgt, labels = vk.synth_community_powerlaw(n, 25, 8, 0.8, 7, 0)
    roles = vk.synth_roles(n, 0.08, 0, 0, 3)
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    scores = np.random.default_rng(1).random((8, n))
    oon, _ = vk.build_reorder(labels, 8, scores)
    ng, r2, l2 = vk.apply_reorder(g, roles, labels, oon)
    noff, ntgt = ng.forward()
    assert ng.symmetric and ng.m == g.m
    deg_old = np.diff(off.astype(np.int64))
    np.testing.assert_array_equal(np.diff(noff.astype(np.int64)), deg_old[oon])
    new_of_old = np.empty(n, np.uint32)
    new_of_old[oon] = np.arange(n, dtype=np.uint32)
    for u in np.random.default_rng(2).integers(0, n, 500):
        row = ntgt[noff[u]:noff[u + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0)
        o = oon[u]
        np.testing.assert_array_equal(np.sort(new_of_old[tgt[off[o]:off[o + 1]]]), row)
    perm = vk.epoch_permutation(r2, l2, 3, 1024, 0, 42)
    s = vk.Sampler(ng, [15, 10, 5], 1024, 1, 42)
    s.run([perm[:1024]], [(0, 3, 0)])
    x = port.expand(CSR(n, noff, ntgt), perm[:1024], [15, 10, 5], 42, 0, 3, 0)
    np.testing.assert_array_equal(s.result(0).all_vertices, x.all_vertices)


@pytest.mark.parametrize("graph,directed", [("pa5000", False), ("dtree13", True)])
def test_baseline_rankings_vs_reference(vk, ref, golden, graph, directed):
    """Fig. 3 baseline rankings (policies.cpp:57-132) on the device: order,
    scores (f64, incl. wPR's dangling mass on the directed tree) and the
    halo's effective alpha bit-identical to the live reference."""
    csr = csr_from(golden("graphs.npz"), graph)
    n = csr.n
    rng = np.random.default_rng(11)
    K = 3
    labels = (np.arange(n) % K).astype(np.uint32)
    roles = np.where(rng.random(n) < 0.4, 0, 1).astype(np.uint8)
    roles[:K] = 0  # every partition has train vertices
    g = (vk.Graph.from_csr(csr.off, csr.tgt, validate=True) if directed
         else vk.Graph.from_csr(csr.off, csr.tgt, undirected=True))
    for k in range(K):
        for L in (1, 2, 3):
            o, s = vk.rank_degree(g, roles, labels, K, k, L)
            eo, es, _ = ref.rank_policy(csr, 0, roles, labels, K, k, L=L)
            np.testing.assert_array_equal(o, eo)
            np.testing.assert_array_equal(s, es)
            o, s = vk.rank_numpaths(g, roles, labels, K, k, L)
            eo, es, _ = ref.rank_policy(csr, 3, roles, labels, K, k, L=L)
            np.testing.assert_array_equal(o, eo)
            np.testing.assert_array_equal(s, es)
        o, s, ea = vk.rank_halo_1hop(g, labels, K, k)
        eo, es, eea = ref.rank_policy(csr, 1, roles, labels, K, k)
        np.testing.assert_array_equal(o, eo)
        np.testing.assert_array_equal(s, es)
        assert ea == eea
        for f1, iters, d in ((2, 5, 0.85), (10, 3, 0.5)):
            o, s = vk.rank_wpr(g, roles, labels, K, k, f1, iters, d)
            eo, es, _ = ref.rank_policy(csr, 2, roles, labels, K, k, f1=f1, iters=iters, damping=d)
            np.testing.assert_array_equal(o, eo)
            np.testing.assert_array_equal(s, es)
    with pytest.raises(vk.ParameterError):
        vk.rank_wpr(g, roles, labels, K, 0, 2, 0)


def _gather_host(vk, plane, sampler, nmb, stream=0):
    view = sampler.view()
    rb = plane.row_bytes
    out_ptr, cnt_ptr = C.c_void_p(), C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(0, nmb * view.all_stride * rb, C.byref(out_ptr)))
    vk.check(vk.lib().vk_device_alloc(0, nmb * 32, C.byref(cnt_ptr)))
    plane.gather(sampler, out_ptr.value, view.all_stride, cnt_ptr.value, stream=stream)
    return out_ptr, cnt_ptr, view.all_stride


def test_gather_wide_rows_exact_row_index(vk, port, golden):
    """fp32 rows of 20001 features (V = 20001 4-byte vectors > 11585): the
    warp's flattened element -> row mapping (umulhi with ceil(2^32/V)) needs
    its fix-up there; rows must still be bit-exact."""
    fx = golden("expand_grid.npz")
    csr = csr_from(golden("graphs.npz"), "pa5000")
    roles, labels = fx["roles"], fx["labels"]
    dim = 20001
    r = _pipeline(vk, port, csr, roles, labels, 4, [3, 2], 16, 0.2, 42, dim, 0, 77, 1)
    for i, (e, k, bi) in enumerate(r["refs"]):
        x = port.expand(csr, r["batches"][i], [3, 2], 42, e, k, bi)
        exp = port.features(77, dim, x.all_vertices)
        got = r["rows"][i].view(np.uint32).reshape(-1, dim)
        np.testing.assert_array_equal(got, exp.view(np.uint32))


def test_two_samplers_gather_on_separate_stream(vk, port, golden):
    """Two samplers alternate on their own streams while every gather runs on
    a third stream with no host synchronisation in between: run i+2 must not
    rewrite the workspace gather i still reads."""
    torch = pytest.importorskip("torch")
    fx = golden("expand_grid.npz")
    csr = csr_from(golden("graphs.npz"), "pa5000")
    roles, labels = fx["roles"], fx["labels"]
    K, b, fan, dim = 4, 64, [15, 10, 5], 64
    n = csr.n
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, b) for k in range(K)])
    totals = np.stack([s.total for s in vk.propagate(g, fan, p0, with_hops=False)])
    plan = vk.build_cache([vk.rank_by_scores(labels, k, totals[k])[0] for k in range(K)], 0.2, n)
    oon, ranges = vk.build_reorder(labels, K, totals)
    plane = vk.FeaturePlane(n, K, dim, labels, oon, ranges)
    for k in range(K):
        plane.load_partition(k, plan.cached[k], feature_seed=5)
    waves = []
    for k in range(K):
        perm = vk.epoch_permutation(roles, labels, k, b, 0, 42)
        waves.append(([perm[i * b:(i + 1) * b] for i in range(2)], [(0, k, i) for i in range(2)]))
    samplers = [vk.Sampler(g, fan, b, 2, 42) for _ in range(2)]
    gs = torch.cuda.Stream()
    outs = []
    for w, (batches, refs) in enumerate(waves):
        s = samplers[w % 2]
        s.run(batches, refs)
        outs.append(_gather_host(vk, plane, s, len(batches), stream=gs.cuda_stream))
    gs.synchronize()
    rb = plane.row_bytes
    for w, (batches, refs) in enumerate(waves):
        out_ptr, cnt_ptr, stride = outs[w]
        for i, (e, k, bi) in enumerate(refs):
            x = port.expand(csr, batches[i], fan, 42, e, k, bi)
            buf = np.zeros(len(x.all_vertices) * rb, np.uint8)
            vk.check(vk.lib().vk_memcpy(buf.ctypes.data, out_ptr.value + i * stride * rb, buf.nbytes, 2))
            np.testing.assert_array_equal(buf.view(np.uint32), port.features(5, dim, x.all_vertices).view(np.uint32).ravel())
        vk.lib().vk_device_free(out_ptr)
        vk.lib().vk_device_free(cnt_ptr)
