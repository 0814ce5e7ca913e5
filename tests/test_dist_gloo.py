"""World-size-2 gloo test of the multi-rank host logic used by bench.py:
per-rank calibration samples are combined with a MAX all-reduce, every rank
fits and solves the plan on its own host, and agree_plan (paper Algorithm 2
line 8, Bcast(m)) verifies the ranks hold the identical plan — and fails
loudly when they do not.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_1912_09268_b200 import dist as D
    from paper_1912_09268_b200 import gradsched as gs

    try:
        D.init("gloo")
        sizes = [4096 * 2 ** k for k in range(12)]
        # rank-dependent jitter: the MAX reduction makes the inputs identical
        times = torch.tensor([8e-6 + s / 600e9 * (1.0 + 0.01 * rank) for s in sizes], dtype=torch.float64)
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
        model = gs.fit_model([gs.CommMeasurement(s, t) for s, t in zip(sizes, times.tolist())])
        trace = gs.load_trace(os.path.join(ROOT, "tests", "golden", "skewed_161.json"))
        trace.forward_time = 5e-3
        for l in trace.layers:
            l.backward_time *= 0.001
        plan = gs.optimal_plan(trace, model)
        digest = D.agree_plan(plan.tags)
        # a rank that solved a different plan must be caught
        bad = list(plan.tags)
        if rank == 1:
            bad[-1] = gs.LayerTag.kMerged if bad[-1] == gs.LayerTag.kNormal else gs.LayerTag.kNormal
        try:
            D.agree_plan(bad)
            caught = False
        except RuntimeError:
            caught = True
        q.put((rank, digest, caught, plan.merged_count()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), False, -1))


def test_two_ranks_agree_on_the_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0][1] == res[1][1], res
    assert len(res[0][1]) == 64
    assert res[0][2] and res[1][2]
    assert res[0][3] == res[1][3] and res[0][3] > 0
