"""Probe: the steps of test_plain_allreduce_p1_is_identity_and_calibration_fits
with progress prints (tools only)."""
import faulthandler
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(60, exit=True)
import torch  # noqa: E402

from paper_1912_09268_b200 import runtime as rt  # noqa: E402

torch.cuda.set_device(0)
comm = rt.Comm(0, 1, 0, 64 << 20)
x = torch.randn(1000003, device="cuda")
y = x.clone()
comm.allreduce_(y)
torch.cuda.synchronize()
print("allreduce ok", torch.equal(x, y), flush=True)
sizes = [4096 << k for k in range(0, 13, 2)]
model, meas = rt.calibrated_model(comm, sizes, warmup=2, reps=5)
print("calibrate ok", model, flush=True)
for s in sizes:
    m = comm.calibrate_engine([s], warmup=1, reps=3)
    print("engine", s, m[0].time_sec * 1e6, "us", flush=True)
