"""TEST INFRASTRUCTURE ONLY (see oracle/README.md).

Regenerates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libvipkit_ref.so, built from /root/reference/proj/src by
`make -C oracle`). The reference ships no golden vectors for the sampler
(SURVEY §8c), so these fixtures pin the reference's own outputs on small,
seeded inputs that mirror its test fixtures:

  * rng.npz        mix64 / SeedSpec::key / RngStream draws incl. power-of-two bounds
  * graphs.npz     generate_synthetic outputs (path, star, tree, grid, PA, uniform)
  * expand_*.npz   epoch_minibatches + expand (frontiers, all_vertices, MFG)
  * vip_*.npz      initial_probs + propagate (hop vectors, totals)
  * policy.npz     rank_by_scores, build_cache, simulate tallies, build_reorder

Usage:  python oracle/make_golden.py   (run where /root/reference exists)
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name), **arrays)


def csr_arrays(prefix, g):
    return {f"{prefix}_off": g.off, f"{prefix}_tgt": g.tgt, f"{prefix}_roff": g.rev_off,
            f"{prefix}_rtgt": g.rev_tgt}


def main():
    R = O.ref()
    R.set_threads(1)

    # ---- rng (rng.hpp:9-74)
    xs = np.array([0, 1, 2, 42, 0xB2, 2**63, 2**64 - 1, 0x9E3779B97F4A7C15], np.uint64)
    mixes = np.array([R.mix64(int(x)) for x in xs], np.uint64)
    keys = np.array([R.seed_key(42, [0xB2, 0, 0, 0, 1, v]) for v in range(16)]
                    + [R.seed_key(42, [0xB1, 3, 5])] + [R.seed_key(7, [0xA1, 1])], np.uint64)
    bounds = [0, 1, 2, 3, 5, 7, 16, 1024, 1000003, 2**32 - 1, 2**32, 2**40 + 7, 2**63]
    draws = np.stack([R.stream_draws(12345 + i, b, 64) for i, b in enumerate(bounds)])
    save("rng.npz", xs=xs, mixes=mixes, keys=keys, bounds=np.array(bounds, np.uint64), draws=draws)

    # ---- graphs (graph.cpp:139-245)
    specs = {"path3": ("path", 3, 2, 0), "star5": ("star", 5, 2, 0), "tree13": ("tree", 13, 3, 0),
             "grid20": ("grid", 20, 4, 0), "pa400": ("pa", 400, 4, 15), "pa150": ("pa", 150, 3, 13),
             "pa120": ("pa", 120, 3, 5), "uni200": ("uniform", 200, 4, 8),
             "uni300": ("uniform", 300, 4, 77), "pa5000": ("pa", 5000, 8, 7)}
    arrays = {}
    for name, (kind, n, d, s) in specs.items():
        arrays.update(csr_arrays(name, R.generate(kind, n, d, s)))
    # directed 13-vertex ternary tree (test_vip.cpp:79-81)
    dtree = R.from_edges(13, [((v - 1) // 3, v) for v in range(1, 13)], undirected=False)
    arrays.update(csr_arrays("dtree13", dtree))
    save("graphs.npz", **arrays)

    # ---- expand on the SmallSetup fixture (test_commsim.cpp:20-28)
    g = R.generate("pa", 400, 4, 15)
    roles = R.make_roles(400, 0.25, 0, 0, 6)
    labels = R.partition(g, roles, 4, "bfs_greedy", 2)
    out = {"roles": roles, "labels": labels, "fanouts": np.array([4, 3], np.uint32), "seed": 77,
           "b": 16}
    idx = 0
    for e in range(2):
        for k in range(4):
            perm = R.epoch_permutation(roles, labels, k, 16, e, 77, K=4)
            out[f"perm_e{e}_k{k}"] = perm
            for i in range(0, (len(perm) + 15) // 16):
                x = R.expand(g, perm[i * 16:(i + 1) * 16], [4, 3], 77, e, k, i)
                p = f"mb{idx}"
                out[p + "_ref"] = np.array([e, k, i], np.uint64)
                out[p + "_batch"] = x.batch
                out[p + "_all"] = x.all_vertices
                for h in range(2):
                    out[f"{p}_f{h + 1}"] = x.frontier[h]
                    out[f"{p}_ip{h + 1}"] = x.indptr[h]
                    out[f"{p}_ed{h + 1}"] = x.edges[h]
                idx += 1
    out["nmb"] = idx
    save("expand_small.npz", **out)

    # ---- expand on the acceptance grid graph (acceptance.cpp:72-80), (15,10,5), b=64
    g = R.generate("pa", 5000, 8, 7)
    roles = R.make_roles(5000, 0.2, 0, 0, 3)
    labels = R.partition(g, roles, 4, "bfs_greedy", 1)
    out = {"roles": roles, "labels": labels, "fanouts": np.array([15, 10, 5], np.uint32),
           "seed": 42, "b": 64}
    idx = 0
    for k in range(4):
        perm = R.epoch_permutation(roles, labels, k, 64, 0, 42, K=4)
        for i in (0, 1, (len(perm) + 63) // 64 - 1):  # includes the ragged last batch
            x = R.expand(g, perm[i * 64:(i + 1) * 64], [15, 10, 5], 42, 0, k, i)
            p = f"mb{idx}"
            out[p + "_ref"] = np.array([0, k, i], np.uint64)
            out[p + "_batch"] = x.batch
            out[p + "_all"] = x.all_vertices
            for h in range(3):
                out[f"{p}_f{h + 1}"] = x.frontier[h]
                out[f"{p}_ip{h + 1}"] = x.indptr[h]
                out[f"{p}_ed{h + 1}"] = x.edges[h]
            idx += 1
    out["nmb"] = idx
    save("expand_grid.npz", **out)

    # ---- VIP (vip.cpp:25-83)
    vip = {}
    hop, tot = R.propagate(R.generate("path", 3), [1, 1], np.array([1.0, 0, 0]))
    vip.update(path3_hop=hop, path3_total=tot)
    g150 = R.generate("pa", 150, 3, 13)
    p0 = np.zeros(150)
    p0[5] = 1.0
    hop, tot = R.propagate(g150, [1000, 1000, 1000], p0)
    vip.update(sat_hop=hop, sat_total=tot)
    p0 = np.zeros(13)
    p0[0] = 1.0
    hop, tot = R.propagate(dtree, [2, 2], p0)
    vip.update(dtree_hop=hop, dtree_total=tot)
    for k in range(4):
        p0 = R.initial_probs(roles, labels, 4, k, 64)
        hop, tot = R.propagate(g, [15, 10, 5], p0)
        vip[f"grid_p0_{k}"] = p0
        vip[f"grid_hop_{k}"] = hop
        vip[f"grid_total_{k}"] = tot
    save("vip.npz", **vip)

    # ---- policies / commsim / reorder on SmallSetup
    g = R.generate("pa", 400, 4, 15)
    roles = R.make_roles(400, 0.25, 0, 0, 6)
    labels = R.partition(g, roles, 4, "bfs_greedy", 2)
    pol = {"roles": roles, "labels": labels}
    orders, totals = [], []
    for k in range(4):
        _, tot = R.propagate(g, [4, 3], R.initial_probs(roles, labels, 4, k, 16))
        o, s = R.rank_by_scores(labels, 4, k, tot)
        pol[f"total_{k}"] = tot
        pol[f"order_{k}"] = o
        pol[f"score_{k}"] = s
        orders.append(o)
        totals.append(tot)
    for a in (0.0, 0.1, 0.15, 3.0):
        cached, bits = R.build_cache(orders, a, 400)
        tag = str(a).replace(".", "p")
        pol[f"bits_{tag}"] = bits
        pol[f"cells_{tag}"] = R.simulate(g, roles, labels, 4, [4, 3], 16, 3, 77, cached)
    oon, ranges = R.build_reorder(labels, 4, np.stack(totals))
    pol.update(old_of_new=oon, ranges=ranges)
    # tie order fixture (test_policies.cpp:160-173)
    o, _ = R.rank_by_scores(np.array([0, 1, 1, 1], np.uint32), 2, 0, np.full(4, 5.0))
    pol["tie_order"] = o
    save("policy.npz", **pol)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
