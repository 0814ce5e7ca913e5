"""Probe: does the persistent comm engine see the replay kernels' ready
signals? Prints engine state while one iteration runs (tools only)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_09268_b200 import _lib  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

torch.cuda.set_device(0)
counts = [4096, 1000, 70000, 5]
tr = gs.trace_from_arrays(counts, [1e-4, 2e-4, 3e-4, 1e-4], 1e-3)
comm = rt.Comm(0, 1, 0, 16 << 20)
g = [torch.ones(c, device="cuda") for c in counts]
w = [torch.zeros(c, device="cuda") for c in counts]
dp = rt.DevicePlan(comm, g, w, gs.MergePlan.all_normal(4))
for ctas in [int(x) for x in os.environ.get("CTAS", "8,-1").split(",")]:
    pipe = rt.Pipeline(dp, tr, 1.0, record_group_times=True, engine_ctas=ctas)
    pipe.launch(1)
    st = (C.c_uint32 * 4)()
    ck = (C.c_uint64 * 2)()
    for i in range(8):
        _lib.mgw_pipeline_debug(pipe.handle, st, ck)
        print(f"ctas={ctas} t={i * 0.25:.2f}s ready={st[0]} iter={st[1]} exit={st[2]} timeout={st[3]} clock={ck[0]},{ck[1]}", flush=True)
        if st[1] >= 1:
            break
        time.sleep(0.25)
    torch.cuda.synchronize()
    print("group ms", pipe.group_times_ms(), "iter ms", pipe.run(3), flush=True)
    pipe.close()
