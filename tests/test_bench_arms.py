"""CPU: bench.py's reference arm runs the reference's own CPU path without
loading the product, and the oracle's restatement of the bench graph recipe
is bit-identical to the product generator it stands in for."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_generator_matches_product(port):
    from paper_2305_03152_b200 import vipkit as vk
    for n, d, c, p_in, seed in ((5000, 4, 3, 0.8, 7), (120000, 12, 8, 0.95, 3), (2, 1, 1, 1.0, 0)):
        o1, t1, l1 = port.synth_community_powerlaw(n, d, c, p_in, seed, threads=3)
        o2, t2, l2 = vk.synth_community_powerlaw(n, d, c, p_in, seed, 0)
        np.testing.assert_array_equal(o1, o2)
        np.testing.assert_array_equal(t1, t2)
        np.testing.assert_array_equal(l1, l2)


def test_cpu_gather_restatement(port):
    table = port.feature_table(99, 24, 1000, fp16=True, threads=2)
    ids = np.random.default_rng(0).integers(0, 1000, 5000).astype(np.uint32)
    np.testing.assert_array_equal(port.gather_rows(table, ids, threads=3), table[ids])
    np.testing.assert_array_equal(table[ids].view(np.uint16), port.features(99, 24, ids, fp16=True).view(np.uint16))


SCRIPT = r"""
import json, os, sys
sys.path.insert(0, ROOT)
import bench
cfg = dict(workload="tiny", n=20000, d=6, K=2, p_in=0.8, train=0.1, dim=16, dtype=1, alpha=0.1,
           fanouts=(5, 3), b=64, wave=8)
class A: gpus = 1; steps = 2; warmup = 3; wave = 8
bench.run_reference(A, cfg)
maps = open("/proc/self/maps").read()
print(json.dumps({"product_module": any(m.startswith("paper_2305_03152_b200") for m in sys.modules),
                  "product_so": "libvipkit_b200" in maps, "ref_so": "libvipkit_ref" in maps}))
"""


def test_reference_arm_is_product_free():
    from oracle import oracle as O
    if not O.ref_available():
        import pytest
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "-c", "ROOT=%r\n" % ROOT + SCRIPT], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    line, probe = lines[0], lines[1]
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
    assert not probe["product_module"] and not probe["product_so"] and probe["ref_so"]
