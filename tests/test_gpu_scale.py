"""GPU, at the benchmarked scale:

* VIP in float-storage mode -- the mode every bench config runs in (n*C*8 B
  > 64 MB) -- on the bench's C3 graph with all 8 partition columns in one
  pass, against the unmodified reference propagate (vip.cpp:37-83): 1e-5
  relative, exact zero pattern; and float mode on rows past the split
  threshold (in-degree > 32768).
* C4 (ogbn-papers100M-shaped, 111 M vertices / 3.3 B CSR slots, fp16 128-d
  rows) in the bench's own wave of 64 minibatches: every minibatch checked for
  the SURVEY §8a invariants, identical between the sparse (bucket, default)
  and dense (bitmap) frontier representations, and 4 minibatches bit-exact
  against the oracle (frontiers, MFG, relabel maps, all_vertices, gathered
  rows, local/cache/miss tallies)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.oracle import CSR
from test_gpu_fullsize import assert_bit_exact, assert_invariants

pytestmark = pytest.mark.gpu


def close(a, b):
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-300)
    assert np.array_equal(a == 0, b == 0)


def test_vip_c3_float_storage_8_columns_vs_reference(vk, ref):
    n, K, fan, b = 2_449_029, 8, [15, 10, 5], 1024
    off, tgt, labels = vk.synth_community_powerlaw(n, 25, K, 0.8, 7, 0)
    roles = vk.synth_roles(n, 0.08, 0, 0, 3)
    assert n * K * 8 > 64 << 20  # the automatic float-storage regime
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, b) for k in range(K)])
    res = vk.propagate(g, fan, p0)
    csr = CSR(n, off, tgt)
    ref.set_threads(os.cpu_count() or 1)
    ref.graph_symmetric(csr)
    for k in range(K):
        np.testing.assert_array_equal(ref.initial_probs(roles, labels, K, k, b), p0[k])
        hop, tot = ref.propagate(csr, fan, p0[k])
        for h in range(3):
            close(res[k].hop[h], hop[h])
        close(res[k].total, tot)
    ref.release(csr)


def test_vip_float_storage_split_rows_vs_reference(vk, ref, port, float_storage):
    """Rows with in-degree > 32768 take the chunked (split) reduction; in
    float storage (forced: this graph is below the automatic threshold) with
    8 columns, against the reference."""
    n = 150_000
    rng = np.random.default_rng(3)
    # three hubs adjacent to almost everything, plus a sparse random part
    hubs = np.array([0, 1, 2], np.uint32)
    src = np.concatenate([np.repeat(hubs, n - 3), rng.integers(3, n, 200_000).astype(np.uint32)])
    dst = np.concatenate([np.tile(np.arange(3, n, dtype=np.uint32), 3), rng.integers(3, n, 200_000).astype(np.uint32)])
    csr = ref.from_edges(n, np.stack([src, dst], 1), True)
    assert np.diff(csr.rev_off.astype(np.int64)).max() > 32768
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    p0 = np.zeros((8, n))
    for c in range(8):
        p0[c, rng.choice(n, 5000 * (c + 1), replace=False)] = rng.random() * 0.9 + 0.05
    res = vk.propagate(g, [10, 5, 3], p0)
    for c in range(8):
        hop, tot = ref.propagate(csr, [10, 5, 3], p0[c])
        for h in range(3):
            close(res[c].hop[h], hop[h])
        close(res[c].total, tot)


def test_c4_wave_sample_and_gather(vk, port):
    n, d, K, b, fan, dim, seed, fseed, M = 111_059_956, 15, 8, 1024, [15, 10, 5], 128, 42, 1234, 64
    off, tgt, labels = vk.synth_community_powerlaw(n, d, K, 0.8, 7, 0)
    roles = vk.synth_roles(n, 0.011, 0, 0, 3)
    csr = CSR(n, off, tgt)
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    # the bench's VIP plan: all partitions in one pass, alpha = 0.32
    p0 = np.stack([vk.initial_probs(roles, labels, k, b) for k in range(K)])
    totals = np.stack([x.total for x in vk.propagate(g, fan, p0, with_hops=False)])
    del p0
    plan = vk.build_cache([vk.rank_by_scores(labels, k, totals[k])[0] for k in range(K)], 0.32, n)
    oon, ranges = vk.build_reorder(labels, K, totals)
    del totals
    plane = vk.FeaturePlane(n, K, dim, labels, oon, ranges, dtype=1)
    for k in range(K):
        plane.load_partition(k, plan.cached[k], feature_seed=fseed)
    batches, refs = [], []
    for k in range(K):
        perm = vk.epoch_permutation(roles, labels, k, b, 0, seed)
        for i in range(M // K):
            batches.append(perm[i * b:(i + 1) * b])
            refs.append((0, k, i))
    s = vk.Sampler(g, fan, b, M, seed)  # automatic: sparse frontiers at this scale
    dense = vk.Sampler(g, fan, b, M, seed, frontier="dense")
    s.run(batches, refs)
    dense.run(batches, refs)
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
        exact = {0, 21, 42, M - 1}
        for i in range(M):
            r = s.result(i)
            q = dense.result(i)
            np.testing.assert_array_equal(r.all_vertices, q.all_vertices)
            for h in range(3):
                np.testing.assert_array_equal(r.frontier[h], q.frontier[h])
                np.testing.assert_array_equal(r.mfg_indptr[h], q.mfg_indptr[h])
                np.testing.assert_array_equal(r.mfg_dst[h], q.mfg_dst[h])
            for h in range(4):
                np.testing.assert_array_equal(r.all_index[h], q.all_index[h])
            assert_invariants(r, off, tgt, fan, rng)
            e, k, bi = refs[i]
            assert tuple(int(c) for c in counts[i][:3]) == port.classify(r.all_vertices, labels, k,
                                                                         plan.member_bits[k])
            if i in exact:
                x = port.expand(csr, batches[i], fan, seed, e, k, bi)
                assert_bit_exact(r, x, len(fan))
                rows = np.zeros((len(r.all_vertices), dim), np.float16)
                vk.check(vk.lib().vk_memcpy(rows.ctypes.data, out.value + i * view.all_stride * rb,
                                            rows.nbytes, 2))
                exp = port.features(fseed, dim, r.all_vertices, fp16=True)
                np.testing.assert_array_equal(rows.view(np.uint16), exp.view(np.uint16))
    finally:
        vk.lib().vk_device_free(out)
        vk.lib().vk_device_free(cnt)
