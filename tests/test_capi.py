"""CPU: the C-ABI library loads, exports every symbol include/vipkit_b200.h
declares, and its host-side entry points (no GPU needed) match the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "vipkit_b200.h")).read()
    return sorted(set(re.findall(r"VK_API\s+[\w\s\*]+?\b(vk_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2305_03152_b200 import vipkit
    L = vipkit.lib()
    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_cpp_mirror_header_names_only_declared_symbols():
    path = os.path.join(ROOT, "include", "vipkit_b200", "vipkit.hpp")
    if not os.path.exists(path):
        pytest.skip("C++ mirror header not written yet")
    txt = open(path).read()
    used = set(re.findall(r"\b(vk_[a-z_0-9]+)\s*\(", txt))
    assert used <= set(header_symbols()), used - set(header_symbols())


def test_no_device_is_reported_not_faked():
    from paper_2305_03152_b200 import vipkit
    n = vipkit.device_count()
    assert n >= 0
    if n == 0:  # CPU box: every compute call must fail loudly, never fall back
        with pytest.raises(vipkit.VipkitError):
            vipkit.Graph.from_csr(np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32),
                                  undirected=True)


def test_status_names_match_reference_error_types():
    from paper_2305_03152_b200 import vipkit
    L = vipkit.lib()
    names = {c: L.vk_status_name(c).decode() for c in range(1, 10)}
    assert names == {1: "parse_error", 2: "range_error", 3: "parameter_error", 4: "format_error",
                     5: "partition_error", 6: "sampling_error", 7: "config_error",
                     8: "shape_error", 9: "io_error"}


def test_host_entry_points_match_oracle(port):
    from paper_2305_03152_b200 import vipkit
    n = 2000
    roles = vipkit.synth_roles(n, 0.3, 0.1, 0.1, 11)
    np.testing.assert_array_equal(roles, port.make_roles(n, 0.3, 0.1, 0.1, 11))
    labels = (np.arange(n) * 7 % 3).astype(np.uint32)
    for k in range(3):
        np.testing.assert_array_equal(vipkit.initial_probs(roles, labels, k, 64),
                                      port.initial_probs(roles, labels, 3, k, 64))
        for e in range(3):
            np.testing.assert_array_equal(vipkit.epoch_permutation(roles, labels, k, 64, e, 42),
                                          port.epoch_permutation(roles, labels, k, 64, e, 42))
    for a, K in [(0.16, 4), (0.2, 8), (0.1, 2), (0.0, 1), (3.0, 4)]:
        assert vipkit.cache_capacity(a, 2449029, K) == port.cache_capacity(a, 2449029, K)


def test_host_errors_map_to_reference_types():
    from paper_2305_03152_b200 import vipkit
    with pytest.raises(vipkit.ParameterError):
        vipkit.cache_capacity(-0.5, 100, 4)
    with pytest.raises(vipkit.ParameterError):
        vipkit.epoch_permutation(np.zeros(10, np.uint8), np.zeros(10, np.uint32), 0, 0, 0, 1)
    with pytest.raises(vipkit.SamplingError):
        vipkit.epoch_permutation(np.full(10, 3, np.uint8), np.zeros(10, np.uint32), 0, 4, 0, 1)
    with pytest.raises(vipkit.SamplingError):
        vipkit.initial_probs(np.full(10, 3, np.uint8), np.zeros(10, np.uint32), 0, 1)
    with pytest.raises(vipkit.ParameterError):
        vipkit.synth_roles(10, 0.8, 0.3)


def test_synthetic_generator_is_canonical_and_deterministic():
    from paper_2305_03152_b200 import vipkit
    off, tgt, lab = vipkit.synth_community_powerlaw(20000, 6, 4, 0.8, 5, threads=3)
    off2, tgt2, lab2 = vipkit.synth_community_powerlaw(20000, 6, 4, 0.8, 5, threads=7)
    np.testing.assert_array_equal(off, off2)
    np.testing.assert_array_equal(tgt, tgt2)
    np.testing.assert_array_equal(lab, lab2)
    n = 20000
    assert off[0] == 0 and off[-1] == len(tgt)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off).astype(np.int64))
    assert np.all(src != tgt)                                  # no self loops
    rows_sorted = np.all((np.diff(tgt.astype(np.int64)) > 0) | (np.diff(src) != 0))
    assert rows_sorted                                          # strictly increasing rows
    key = src * n + tgt
    rkey = tgt.astype(np.int64) * n + src
    np.testing.assert_array_equal(np.sort(key), np.sort(rkey))  # symmetric
    assert np.bincount(lab).min() == n // 4                     # balanced communities
    intra = (lab[src] == lab[tgt]).mean()
    assert intra > 0.7                                          # partitionable structure
