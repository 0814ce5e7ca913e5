"""Single-GPU loopback probe of the fused group kernel (tools only; for ncu):
P emulated ranks in one cooperative launch, one merge group of SIZE_MB."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

P = int(os.environ.get("P", "2"))
n = (int(os.environ.get("SIZE_MB", "64")) << 20) // 4
algo = os.environ.get("ALGO", "twoshot")
iters = int(os.environ.get("ITERS", "5"))
torch.cuda.set_device(0)
gdt = torch.bfloat16 if os.environ.get("DTYPE") == "bf16" else torch.float32
grads = [[torch.rand(n, device="cuda").to(gdt)] for _ in range(P)]
weights = [[torch.rand(n, device="cuda")] for _ in range(P)]
comm = rt.Comm.create_loopback(P, 0, 4 * n)
dp = rt.DevicePlan(comm, grads, weights, gs.MergePlan.all_merged(1))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    dp.group_allreduce(0, 0.01, rt.SGD, algo)
torch.cuda.synchronize()
e0.record()
for _ in range(iters):
    dp.group_allreduce(0, 0.01, rt.SGD, algo)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / iters * 1e3
print(f"loopback P={P} {algo} {n * 4 >> 20} MiB/rank: {us:.1f} us/launch, "
      f"local HBM {P * n * 4 * (6 if algo == 'twoshot' else 5) / us / 1e3:.0f} GB/s (approx)")
dp.close()
comm.close()
