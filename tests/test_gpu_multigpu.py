"""GPU (>= 2 devices): multi-GPU gather parity. Each rank owns partitions
k = rank (mod N) and reads the others' rows over NVLink inside the gather
kernel; rows/tallies bit-exact vs the oracle (tests/multigpu_parity.py)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_two_gpu_gather_parity(vk):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run via gpurun --gpus 2)")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(ROOT, "tests", "multigpu_parity.py")],
                       capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert r.stdout.count(": ok") == 2
