"""HBM roofline probe of the rank-local kernels (tools only; for ncu too):
pack (2S), unpack+SGD (3S) and the P=1 fused group kernel (3S) on one merge
group of LAYERS x LAYER_MB, CUDA-event timed, L2 flushed between reps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

L = int(os.environ.get("LAYERS", "64"))
n = (int(os.environ.get("LAYER_MB", "4")) << 20) // 4
reps = int(os.environ.get("REPS", "10"))
torch.cuda.set_device(0)
grads = [torch.rand(n, device="cuda") for _ in range(L)]
weights = [torch.rand(n, device="cuda") for _ in range(L)]
S = 4 * n * L
comm = rt.Comm(0, 1, 0, S + (1 << 20))
dp = rt.DevicePlan(comm, grads, weights, gs.MergePlan.all_merged(L))
merge = torch.empty(n * L, device="cuda")
flush = torch.empty(512 << 20 >> 2, device="cuda")
peak = None
try:
    import json
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass


def timed(fn):
    if reps == 0:  # one launch each (ncu capture)
        fn()
        torch.cuda.synchronize()
        return float("nan")
    ts = []
    for r in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


for name, fn, nbytes in [
    ("pack (read grads, write merge buffer)", lambda: dp.pack(0, 0.5, merge), 2 * S),
    ("unpack+SGD (read reduced, read W, write W)", lambda: dp.unpack_sgd(0, merge, 0.01), 3 * S),
    ("fused group kernel P=1 (read grad, read W, write W)", lambda: dp.group_allreduce(0, 0.01, rt.SGD), 3 * S),
]:
    t = timed(fn)
    gbs = nbytes / t / 1e9
    frac = f"  {gbs / peak:.2f} of {peak:.0f} GB/s" if peak else ""
    print(f"{name:55s} S={S >> 20} MiB  {t * 1e6:8.1f} us  {gbs:7.1f} GB/s{frac}", flush=True)
dp.close()
comm.close()
