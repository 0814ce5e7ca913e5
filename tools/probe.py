"""Latency probe: calibration of the fused kernel at P=1 for a few sizes
plus back-to-back launches, for ncu launch lists (tools only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_09268_b200 import runtime as rt  # noqa: E402

torch.cuda.set_device(0)
comm = rt.Comm(0, 1, 0, 64 << 20)
sizes = [4096, 65536, 1 << 20, 16 << 20]
meas = comm.calibrate(sizes, warmup=2, reps=int(os.environ.get("REPS", "10")))
for m in meas:
    print(f"{m.size_bytes} {m.time_sec * 1e6:.3f} us")
comm.close()
