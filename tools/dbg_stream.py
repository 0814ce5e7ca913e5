"""Debug probe (tools only): stream-protocol fused group all-reduce in
loopback vs the C oracle on RAGGED layers; prints mismatching layers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pyoracle  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

RAGGED = [1000, 0, 7, 9000, 4096, 13, 20000, 1, 4097, 3, 300000, 5, 1 << 20, 77]


def run(P, algo, proto, max_ctas, epi, iters=1, split=True):
    rng = np.random.default_rng(100 + P)
    counts = RAGGED
    g_np = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    w_np = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    g_dev = [[torch.from_numpy(a.copy()).cuda() for a in per] for per in g_np]
    w_dev = [[torch.from_numpy(a.copy()).cuda() for a in per] for per in w_np]
    plan = gs.MergePlan.all_normal(len(counts)) if split else gs.MergePlan.all_merged(len(counts))
    tags = [int(t) for t in plan.tags]
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    comm.set_oneshot_max(16 * 1024)
    comm.set_protocol(proto)
    comm.set_ll_max(0)
    if max_ctas:
        comm.set_max_ctas(max_ctas)
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    for _ in range(iters):
        for g in reversed(range(dp.n_groups)):
            dp.group_allreduce(g, 0.01, epi, algo)
        pyoracle.allreduce_sgd(g_np, w_np, tags, 0.01, write_grad=bool(epi & rt.WRITE_GRAD))
    torch.cuda.synchronize()
    bad = []
    for r in range(P):
        for l in range(len(counts)):
            a = w_dev[r][l].cpu().numpy()
            if not np.array_equal(a, w_np[r][l]):
                nb = int((a != w_np[r][l]).sum())
                idx = np.nonzero(a != w_np[r][l])[0]
                bad.append((r, l, counts[l], nb, int(idx[0]), int(idx[-1])))
    print(f"P={P} {algo} {proto} ctas={max_ctas} epi={epi} iters={iters} split={split} failed={comm.failed()} "
          f"bad={len(bad)} {bad[:6]}", flush=True)
    dp.close()
    comm.close()


for P in (2, 4, 8):
    for algo in ("twoshot", "oneshot"):
        for ctas in (0, 1, 3):
            run(P, algo, "stream", ctas, rt.SGD)
    run(P, "twoshot", "stream", 0, rt.SGD | rt.WRITE_GRAD, iters=3)
    run(P, "twoshot", "stream", 0, rt.SGD, split=False)
