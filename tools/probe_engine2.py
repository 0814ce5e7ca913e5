"""Probe: engine pipeline over 8 groups of S bytes all ready at t=0, with
state polling (tools only)."""
import ctypes as C
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(100, exit=True)
import torch  # noqa: E402

from paper_1912_09268_b200 import _lib  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

torch.cuda.set_device(0)
comm = rt.Comm(0, 1, 0, 64 << 20)
for S, ctas in [(1 << 20, -1), (4 << 20, 64), (4 << 20, -1), (4 << 20, 300)]:
    n = S // 4
    R = 8
    g = torch.ones(n, device="cuda")
    w = torch.zeros(n, device="cuda")
    tr = gs.trace_from_arrays([n] * R, [0.0] * R, 0.0)
    dp = rt.DevicePlan(comm, [g] * R, [w] * R, gs.MergePlan.all_normal(R))
    pipe = rt.Pipeline(dp, tr, 0.0, record_group_times=True, engine_ctas=ctas)
    st = (C.c_uint32 * 4)()
    ck = (C.c_uint64 * 2)()
    for it in range(3):
        pipe.launch(1)
        t0 = time.time()
        while True:
            _lib.mgw_pipeline_debug(pipe.handle, st, ck)
            if st[1] >= it + 1 or time.time() - t0 > 15:
                break
            time.sleep(0.05)
        print(f"S={S} ctas={ctas} it={it} after {time.time() - t0:.2f}s: ready={st[0]} iter={st[1]} exit={st[2]} "
              f"timeout={st[3]} clk={ck[0] % 10**9},{ck[1] % 10**9}", flush=True)
    torch.cuda.synchronize()
    print("   group us", [round(x * 1e3, 2) for x in pipe.group_times_ms()], flush=True)
    pipe.close()
    dp.close()
