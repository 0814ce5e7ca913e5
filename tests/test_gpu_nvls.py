"""NVLS (switch-reduced) variant on ONE B200: the API's guard rails. The
data path needs a multicast object over distinct GPUs, so its parity runs
in tests/mr_worker.py (nvls_checks: bit-exact vs the oracle's exact-sum
variant at P = 2 / 4 over NVLink); here the single-GPU contract: a loopback
communicator reports NVLS unsupported and a forced NVLS launch fails
loudly instead of falling back.
"""
import pytest
import torch

from paper_1912_09268_b200 import gradsched as gs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_09268_b200 import runtime as rt


def test_loopback_reports_nvls_unsupported_and_forced_nvls_fails_loudly():
    counts = [1000, 4096]
    comm = rt.Comm.create_loopback(2, 0, 4 * rt.padded_elems(counts))
    assert not comm.nvls_supported()
    assert not comm.nvls_ready
    with pytest.raises(gs.Error):
        comm.set_nvls(1 << 20)  # NVLS not set up: refused
    g = [[torch.zeros(c, device="cuda") for c in counts] for _ in range(2)]
    w = [[torch.zeros(c, device="cuda") for c in counts] for _ in range(2)]
    plan = gs.MergePlan([gs.LayerTag(0), gs.LayerTag(1)])
    dp = rt.DevicePlan(comm, g, w, plan)
    with pytest.raises(gs.Error):
        dp.group_allreduce(0, 0.01, rt.SGD, "nvls")
    dp.close()
    comm.close()
