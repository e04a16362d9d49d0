"""GPU: the reference's own unit tests (test_vip/test_sampling/test_policies
cases) re-hosted in C++ against include/vipkit_b200/vipkit.hpp, the drop-in
C++ mirror of the reference API."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_mirror_reference_cases(vk):
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_mirror")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
