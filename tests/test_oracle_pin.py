"""CPU: the C restatement against the live, unmodified reference library
(oracle/_ref) on seeded random cases beyond the committed fixtures."""
import numpy as np
import pytest


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_vs_ref_expand_and_vip(port, ref, seed):
    n = 3000 + 500 * seed
    gr = ref.generate("pa", n, 3 + seed, seed)
    gp = port.generate("pa", n, 3 + seed, seed)
    np.testing.assert_array_equal(gr.tgt, gp.tgt)
    roles = ref.make_roles(n, 0.3, 0.1, 0.1, seed)
    np.testing.assert_array_equal(roles, port.make_roles(n, 0.3, 0.1, 0.1, seed))
    labels = ref.partition(gr, roles, 3, "random", seed)
    fan = [7, 4, 3][: 2 + seed % 2]
    for k in range(3):
        pr = ref.epoch_permutation(roles, labels, k, 50, seed, 100 + seed, K=3)
        np.testing.assert_array_equal(pr, port.epoch_permutation(roles, labels, k, 50, seed, 100 + seed))
        for i in range(0, min(4, (len(pr) + 49) // 50)):
            b = pr[i * 50:(i + 1) * 50]
            xr = ref.expand(gr, b, fan, 100 + seed, seed, k, i)
            xp = port.expand(gp, b, fan, 100 + seed, seed, k, i)
            np.testing.assert_array_equal(xr.all_vertices, xp.all_vertices)
            for h in range(len(fan)):
                np.testing.assert_array_equal(xr.frontier[h], xp.frontier[h])
                np.testing.assert_array_equal(xr.edges[h], xp.edges[h])
                np.testing.assert_array_equal(xr.indptr[h], xp.indptr[h])
        p0 = ref.initial_probs(roles, labels, 3, k, 50)
        hr, tr = ref.propagate(gr, fan, p0)
        hp, tp = port.propagate(gp, fan, p0)
        np.testing.assert_array_equal(hr, hp)
        np.testing.assert_array_equal(tr, tp)
        o1, s1 = ref.rank_by_scores(labels, 3, k, tr)
        o2, s2 = port.rank_by_scores(labels, 3, k, tp)
        np.testing.assert_array_equal(o1, o2)


def test_port_vs_ref_draws_all_bounds(port, ref):
    for i, bound in enumerate([1, 2, 3, 4, 6, 64, 1 << 20, (1 << 32) + 1, (1 << 63) + 5]):
        np.testing.assert_array_equal(port.stream_draws(i, bound, 500), ref.stream_draws(i, bound, 500))
