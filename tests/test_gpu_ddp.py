"""Real-backward integration: autograd hooks mark merge
groups ready for the persistent comm engine while the backward runs; the
engine applies SGD. At P = 1 the result must equal plain PyTorch SGD
(w - lr*g, two roundings) bit-for-bit. Multi-rank: tests/mr_worker.py.
"""
import copy

import numpy as np
import pytest
import torch

from paper_1912_09268_b200 import gradsched as gs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_09268_b200 import runtime as rt
    from paper_1912_09268_b200.ddp import MGWFBP


def _model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 256),
                               torch.nn.ReLU(), torch.nn.Linear(256, 10)).cuda()


@pytest.mark.parametrize("mode", ["engine", "launch"])
@pytest.mark.parametrize("plan_kind", ["wfbp", "merged_pairs", "single"])
def test_real_backward_sgd_matches_pytorch_p1(plan_kind, mode):
    model = _model()
    ref = copy.deepcopy(model)
    L = len(list(model.parameters()))
    if plan_kind == "wfbp":
        plan = gs.MergePlan.all_normal(L)
    elif plan_kind == "single":
        plan = gs.MergePlan.all_merged(L)
    else:
        plan = gs.MergePlan([gs.LayerTag(0 if i % 2 == 0 else 1) for i in range(L)])
    lr = 0.05
    counts = [p.numel() for p in model.parameters()]
    comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
    sync = MGWFBP(model, comm, lr, plan=plan, engine_ctas=8, record_group_times=True, mode=mode, launch_ctas=4)
    gen = torch.Generator(device="cuda").manual_seed(1)
    lr_t = torch.tensor(lr, device="cuda")
    for _ in range(3):
        x = torch.randn(32, 64, device="cuda", generator=gen)
        y = torch.randint(0, 10, (32,), device="cuda", generator=gen)
        sync.begin()
        torch.nn.functional.cross_entropy(model(x), y).backward()
        sync.end()
        ref.zero_grad(set_to_none=False)
        torch.nn.functional.cross_entropy(ref(x), y).backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.copy_(p - lr_t * p.grad)
    torch.cuda.synchronize()
    sync.check()
    for a, b in zip(model.parameters(), ref.parameters()):
        assert torch.equal(a, b)
    if mode == "engine":
        times = sync.group_times_ms()
        assert all(t > 0 for t in times[sync.tail:])  # engine groups (the tail runs full width after join)
    sync.close()
    comm.close()
