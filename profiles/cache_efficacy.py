"""VIP-cache efficacy on the device: the
Fig. 3-style policy x alpha sweep -- VIP against degree, 1-hop halo, weighted
PageRank, number of paths, simulation ("sim", 2 epochs) and the retrospective
oracle -- on C3-shaped community graphs of increasing locality / popularity skew
(p_in = 0.8 and popularity rank U^2: the bench graph; p_in = 0.95; p_in =
0.95 with rank U^4, i.e. fewer, bigger hubs), one evaluation epoch of all 8
partitions.
improvement = misses without cache / misses with it (sweep's metric,
commsim.cpp:235-247). Usage: python profiles/cache_efficacy.py > out.json"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_03152_b200 import vipkit as vk  # noqa: E402

n, d, K, train, b, fan, seed = 2_449_029, 25, 8, 0.08, 1024, [15, 10, 5], 42
alphas = [0.01, 0.05, 0.1, 0.2]
out = {"graph": f"community power-law n={n} d={d} K={K} train={train}", "fanouts": fan, "batch": b,
       "alphas": alphas, "epochs_evaluated": 1, "runs": []}
for p_in, skew in ((0.8, 2.0), (0.95, 2.0), (0.95, 4.0)):
    t0 = time.time()
    off, tgt, labels = vk.synth_community_powerlaw(n, d, K, p_in, 7, 0, skew=skew)
    roles = vk.synth_roles(n, train, 0, 0, 3)
    g = vk.Graph.from_csr(off, tgt, undirected=True)
    p0 = np.stack([vk.initial_probs(roles, labels, k, b) for k in range(K)])
    vip = np.stack([x.total for x in vk.propagate(g, fan, p0, with_hops=False)])
    access = vk.access_counts(g, roles, labels, K, fan, b, 1, seed)
    policies = {
        "vip": lambda k: vk.rank_by_scores(labels, k, vip[k])[0],
        "deg": lambda k: vk.rank_degree(g, roles, labels, K, k, len(fan))[0],
        "1hop": lambda k: vk.rank_halo_1hop(g, labels, K, k)[0],
        "wpr": lambda k: vk.rank_wpr(g, roles, labels, K, k, fan[0])[0],
        "numpaths": lambda k: vk.rank_numpaths(g, roles, labels, K, k, len(fan))[0],
        "sim": lambda k: vk.rank_by_scores(labels, k, vk.empirical_vip(g, roles, labels, K, k, b, fan, 2, seed))[0],
        "oracle": lambda k: vk.rank_by_scores(labels, k, access[k])[0],
    }
    caps = [vk.cache_capacity(a, n, K) for a in alphas]
    run = {"p_in": p_in, "skew": skew, "m_slots": int(len(tgt)), "policies": {}}
    base = None
    for name, rank in policies.items():
        orders = [rank(k) for k in range(K)]
        cached = [o[:max(caps)] for o in orders]
        takes = [[min(c, len(o)) for o in orders] for c in caps]
        cells = vk.simulate(g, roles, labels, K, fan, b, 1, seed, cached, takes=takes)
        miss = [int(cells[a, :, :, 2].sum()) for a in range(len(alphas))]
        if base is None:
            base = int(cells[0, :, :, 1].sum() + cells[0, :, :, 2].sum())  # no-cache misses
        run["policies"][name] = {"misses": miss, "improvement": [base / max(m, 1) for m in miss]}
        print(f"p_in={p_in} skew={skew} {name}: " + " ".join(f"{base / max(m, 1):.3f}" for m in miss), file=sys.stderr)
    run["no_cache_misses"] = base
    run["seconds"] = time.time() - t0
    out["runs"].append(run)
    del g
print(json.dumps(out))
