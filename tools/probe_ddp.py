"""Probe the real-backward engine path step by step (tools only)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_09268_b200 import _lib  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402
from paper_1912_09268_b200.ddp import MGWFBP  # noqa: E402

torch.manual_seed(0)
model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).cuda()
L = len(list(model.parameters()))
comm = rt.Comm(0, 1, 0, 16 << 20)
sync = MGWFBP(model, comm, 0.05, plan=gs.MergePlan.all_normal(L), engine_ctas=int(os.environ.get("CTAS", "8")))
calls = []
orig = sync._hook


def st():
    s = (C.c_uint32 * 4)()
    ck = (C.c_uint64 * 2)()
    _lib.mgw_pipeline_debug(sync.handle, s, ck)
    return list(s)


print("stream", torch.cuda.current_stream(), "pipe", st(), flush=True)
x = torch.randn(32, 64, device="cuda")
y = torch.randint(0, 10, (32,), device="cuda")
sync.begin()
print("after begin", st(), flush=True)
loss = torch.nn.functional.cross_entropy(model(x), y)
loss.backward()
print("after backward: remaining", sync.remaining, st(), flush=True)
sync.end()
ev = torch.cuda.Event()
ev.record()
t0 = time.time()
while not ev.query() and time.time() - t0 < 15:
    time.sleep(0.1)
print("done" if ev.query() else "STUCK", round(time.time() - t0, 2), st(), flush=True)
torch.cuda.synchronize()
sync.check()
print("check ok", flush=True)
