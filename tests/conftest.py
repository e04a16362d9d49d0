"""Shared fixtures. `-m "not gpu"` runs on a CPU-only box; `-m gpu` needs a B200.

The oracle (oracle/) is test infrastructure: these tests use it as the checker
only. The product under test is paper_2305_03152_b200/libvipkit_b200.so.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (B200) and the built CUDA library")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("compiled reference (oracle/_ref) not built here")
    return O.ref()


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name)))
        return cache[name]
    return load


@pytest.fixture(scope="session")
def vk():
    """The product's Python mirror, with a GPU required (fail, don't skip)."""
    from paper_2305_03152_b200 import vipkit
    assert vipkit.device_count() >= 1, "no sm_100 device visible to libvipkit_b200"
    return vipkit


def csr_from(golden_graphs, name):
    from oracle.oracle import CSR
    g = golden_graphs
    return CSR(len(g[name + "_off"]) - 1, g[name + "_off"], g[name + "_tgt"], g[name + "_roff"],
               g[name + "_rtgt"])


@pytest.fixture
def float_storage(vk):
    """Force the VIP hoisted terms into float storage for one test."""
    vk.vip_force_storage(32)
    yield
    vk.vip_force_storage(0)
