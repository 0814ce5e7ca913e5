"""Multi-GPU parity: torchrun 2 (and 4, 8 when present) ranks, one per GPU,
running tests/mr_worker.py (IPC-mapped merge arenas over NVLink, fused
kernel bit-exact vs the oracle, plain all-reduce vs NCCL, pipeline,
calibration). Skipped with fewer than 2 GPUs.
"""
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_multirank_worker(P):
    if not torch.cuda.is_available() or torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + P}", os.path.join(ROOT, "tests", "mr_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert "MULTIRANK OK" in r.stdout
