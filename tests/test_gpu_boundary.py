"""GPU: the remaining reference entry points of the drop-in boundary (SURVEY
§8b B1) against the live reference: sample_neighbors (sampling.cpp:72-92,
stream state included), simulate's SimulateOptions streams (trace and
batch_costs with the GPU-prefix split, commsim.cpp:77-127), and the C++
mirror fed the reference's own files (VCSR, partition labels, roles, VIP
binary)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, csr_from

pytestmark = pytest.mark.gpu


def _mix64(x):
    m = (1 << 64) - 1
    x = (x + 0x9e3779b97f4a7c15) & m
    x = ((x ^ (x >> 30)) * 0xbf58476d1ce4e5b9) & m
    x = ((x ^ (x >> 27)) * 0x94d049bb133111eb) & m
    return x ^ (x >> 31)


def _next_u64(state):
    m = (1 << 64) - 1
    return _mix64((state) & m)  # next_u64 = mix64-finaliser of counter + golden == mix64(counter)


def test_sample_neighbors_vs_reference(vk, ref, golden):
    csr = csr_from(golden("graphs.npz"), "pa5000")
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    deg = np.diff(csr.off.astype(np.int64))
    hubs = np.argsort(-deg)[:20]
    small = np.where(deg <= 3)[0][:20]
    keys = np.random.default_rng(5).permutation(csr.n).astype(np.uint32)
    for v in list(hubs) + list(small) + [0, 17, 4999]:
        for f in (1, 3, 10, 40):
            key = (int(v) * 7919 + f) & ((1 << 64) - 1)
            for sk in (None, keys):
                exp, nxt = ref.sample_neighbors(csr, int(v), f, key, seed_keys=sk)
                got, state = vk.sample_neighbors(g, int(v), f, _mix64(key), seed_keys=sk, offsets=csr.off,
                                                 targets=csr.tgt)
                np.testing.assert_array_equal(got, exp)
                assert _next_u64(state) == nxt  # the stream advanced exactly as the reference's


def _setup(port, ref, n=3000, K=3):
    csr = port.generate("pa", n, 5, 21)
    roles = port.make_roles(n, 0.2, 0, 0, 3)
    labels = (np.arange(n) % K).astype(np.uint32)
    return csr, roles, labels


def test_simulate_batch_costs_vs_reference(vk, port, ref, tmp_path):
    K = 3
    csr, roles, labels = _setup(port, ref, K=K)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True)
    rng = np.random.default_rng(4)
    cached = [np.setdiff1d(rng.choice(csr.n, 300, replace=False), np.where(labels == k)[0]).astype(np.uint32)
              for k in range(K)]
    orders = [rng.permutation(np.where(labels == k)[0]).astype(np.uint32) for k in range(K)]
    for ords, gamma in ((None, 0.0), (orders, 0.37)):
        path = str(tmp_path / "costs.csv")
        ecells = ref.simulate_streams(csr, roles, labels, K, [5, 3], 32, 2, 42, cached, costs_path=path,
                                      orderings=ords, gamma=gamma)
        exp = np.loadtxt(path, delimiter=",", dtype=np.uint64).reshape(-1, 7)
        cells, rows = vk.simulate_batches(g, roles, labels, K, [5, 3], 32, 2, 42, cached, gpu_orderings=ords,
                                          gamma=gamma)
        np.testing.assert_array_equal(cells, ecells)
        np.testing.assert_array_equal(rows, exp)
        if ords is not None:
            assert rows[:, 4].sum() > 0


def test_cpp_mirror_on_reference_files(vk, port, ref, tmp_path):
    """The C++ mirror loads reference-written VCSR / labels / roles / VIP files
    and its simulate(..., SimulateOptions{trace, batch_costs, gpu_orderings})
    writes the reference's CSV rows byte for byte."""
    K = 3
    csr, roles, labels = _setup(port, ref, K=K)
    d = str(tmp_path)
    ref.write_vcsr(csr, os.path.join(d, "graph.vcsr"))
    ref.write_partition_labels(labels, K, os.path.join(d, "labels.txt"))
    ref.write_roles(roles, os.path.join(d, "roles.txt"))
    p0 = ref.initial_probs(roles, labels, K, 0, 32)
    _, total = ref.propagate(csr, [5, 3], p0)
    ref.write_vip_binary(total, os.path.join(d, "vip0.bin"))
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_mirror")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe, "--reference-files", d], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = dict(line.split(" ", 1) for line in r.stdout.strip().splitlines())
    # the same plan / orderings on the reference side
    orders = [ref.rank_by_scores(labels, K, k, total)[0] for k in range(K)]
    cached, _ = ref.build_cache(orders, 0.1, csr.n)
    ords = [np.where(labels == k)[0][::-1].astype(np.uint32) for k in range(K)]
    cells = ref.simulate_streams(csr, roles, labels, K, [5, 3], 32, 2, 42, cached,
                                 trace_path=os.path.join(d, "ref_trace.csv"),
                                 costs_path=os.path.join(d, "ref_costs.csv"), orderings=ords, gamma=0.3)
    assert open(os.path.join(d, "mirror_trace.csv")).read() == open(os.path.join(d, "ref_trace.csv")).read()
    assert open(os.path.join(d, "mirror_costs.csv")).read() == open(os.path.join(d, "ref_costs.csv")).read()
    assert [int(x) for x in out["cells"].split()] == [int(x) for x in cells.ravel()]
    assert open(os.path.join(d, "mirror_vip0.bin"), "rb").read() == open(os.path.join(d, "vip0.bin"), "rb").read()
    assert int(out["train_members0"]) == int(((labels == 0) & (roles == 0)).sum())
    from oracle.oracle import Ref  # noqa: F401  (reference sample_neighbors with the same stream key)
    key = ref.seed_key(7, [1, 2])
    exp, nxt = ref.sample_neighbors(csr, 0, 4, key)
    assert [int(x) for x in out["sample0"].split()] == list(map(int, exp))
    assert int(out["next"]) == nxt
