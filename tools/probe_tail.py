"""Unsynchronised real-backward iterations with a full-width tail group
(tools only; torchrun, P ranks). Prints progress / pipe state, never hangs:
a host watchdog gives up after 30 s."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_09268_b200 import _lib  # noqa: E402
from paper_1912_09268_b200 import dist as D  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402
from paper_1912_09268_b200.ddp import MGWFBP  # noqa: E402

rank, P, local = D.init("nccl")
torch.cuda.set_device(local)
torch.manual_seed(0)
width = int(os.environ.get("WIDTH", "256"))
layers = [torch.nn.Linear(width, width) for _ in range(int(os.environ.get("DEPTH", "4")))]
model = torch.nn.Sequential(*layers).cuda()
L = len(list(model.parameters()))
counts = [p.numel() for p in model.parameters()]
comm = rt.Comm(rank, P, local, 4 * rt.padded_elems(counts) + (1 << 20))
plan = gs.MergePlan.all_normal(L)
sync = MGWFBP(model, comm, 0.01, plan=plan, engine_ctas=8, tail_groups=int(os.environ.get("TAIL", "1")))
x = torch.randn(64, width, device="cuda")


def st():
    s = (C.c_uint32 * 4)()
    ck = (C.c_uint64 * 2)()
    _lib.mgw_pipeline_debug(sync.handle, s, ck)
    return list(s)


for k in range(int(os.environ.get("ITERS", "10"))):
    sync.begin()
    model(x).square().mean().backward()
    sync.end()
    if os.environ.get("SYNC"):
        torch.cuda.synchronize()
ev = torch.cuda.Event()
ev.record()
t0 = time.time()
while not ev.query() and time.time() - t0 < 30:
    time.sleep(0.1)
print(f"[rank {rank}]", "done" if ev.query() else "STUCK", round(time.time() - t0, 2), st(), flush=True)
if ev.query():
    sync.check()
    print(f"[rank {rank}] check ok", flush=True)
os._exit(0)
