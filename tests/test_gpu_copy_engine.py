"""Copy-engine mode (mgw_ce_*, runtime.CopyEngine) on ONE B200 in loopback:
P emulated ranks, each group's gradients copied into the peers' arenas by
DMA when marked ready, one full-width reduce + SGD after the "backward".
Parity: bit-exact vs the CPU oracle (rank-order fp32 sum, x 1/P per source,
SGD with two roundings) — the same arithmetic as the fused kernels, so the
reference semantics (Eq. 2) are unchanged."""
import numpy as np
import pytest
import torch

from oracle import pyoracle
from paper_1912_09268_b200 import gradsched as gs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_09268_b200 import runtime as rt

RAGGED = [1000, 0, 7, 9000, 4096, 13, 20000, 1, 4097, 3, 300000, 5, 1 << 20, 77]


def _flat(counts, arrays, dtype=torch.float32):
    """One flat buffer per rank in the merge layout (16-byte aligned layer
    starts) and per-layer views into it."""
    offs = [0]
    for c in counts:
        offs.append(offs[-1] + ((c + 3) & ~3))
    bufs, views = [], []
    for per in arrays:
        # exactly to the last element (no tail padding: the copies must not read past it)
        b = torch.zeros(max(offs[-2] + counts[-1], 4), dtype=dtype, device="cuda")
        for l, a in enumerate(per):
            b[offs[l]:offs[l] + counts[l]] = torch.from_numpy(a)
        bufs.append(b)
        views.append([b[offs[l]:offs[l] + counts[l]] for l in range(len(counts))])
    return bufs, views


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("merged", [False, True])
@pytest.mark.parametrize("tail", [0, 1, "1-overlap"])
def test_copy_engine_bit_exact(P, merged, tail):
    """3 iterations; with tail = 1 the last-ready group goes through the
    fused full-width kernel after the backward, the rest through the copy
    engines."""
    rng = np.random.default_rng(900 + P)
    counts = RAGGED
    g_np = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    w_np = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    gbufs, g_dev = _flat(counts, g_np)
    w_dev = [[torch.from_numpy(a.copy()).cuda() for a in per] for per in w_np]
    tr = gs.trace_from_arrays(counts, list(rng.uniform(1e-5, 1e-4, len(counts))), 1e-4)
    plan = gs.optimal_plan(tr, gs.AllReduceModel(2e-5, 1e-12)) if merged else gs.MergePlan.all_normal(len(counts))
    tags = [int(t) for t in plan.tags]
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    overlap = tail == "1-overlap"
    tail = 1 if overlap else tail
    ce = rt.CopyEngine(dp, 0.01)
    ce.set_tail(tail)
    if overlap and not ce.signals_without_sm:
        pytest.skip("no stream memory operations: the tail must follow join()")
    s = torch.cuda.current_stream()
    for it in range(3):
        # a new "backward" each iteration: fresh gradients, groups ready in backward order
        if it:
            for r in range(P):
                for l, c in enumerate(counts):
                    g_np[r][l] = rng.uniform(-1, 1, c).astype(np.float32)
                    g_dev[r][l].copy_(torch.from_numpy(g_np[r][l]))
        ce.begin(s)
        for g in reversed(range(dp.n_groups)):
            ce.mark_ready(g, s)
        if not overlap:
            ce.join(s)
        for g in reversed(range(tail)):  # after the join unless the signals need no SM
            dp.group_allreduce(g, 0.01, rt.SGD, "auto", s)
        if overlap:
            ce.join(s)
        pyoracle.allreduce_sgd(g_np, w_np, tags, 0.01)
    torch.cuda.synchronize()
    ce.check()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    assert not comm.failed()
    ce.close()
    dp.close()
    comm.close()


def test_copy_engine_rejects_non_flat_gradients():
    counts = [100, 200]
    comm = rt.Comm.create_loopback(2, 0, 4 * rt.padded_elems(counts))
    g = [[torch.zeros(c, device="cuda") for c in counts] for _ in range(2)]  # separate allocations
    w = [[torch.zeros(c, device="cuda") for c in counts] for _ in range(2)]
    dp = rt.DevicePlan(comm, g, w, gs.MergePlan.all_normal(2))
    with pytest.raises(gs.ValidationError, match="flat buffer"):
        rt.CopyEngine(dp, 0.01)
    dp.close()
    comm.close()


def test_copy_engine_calibration_is_monotone():
    comm = rt.Comm.create_loopback(2, 0, 64 << 20)
    meas = comm.calibrate_ce([4096, 1 << 20, 16 << 20, 64 << 20], warmup=2, reps=5)
    ts = [m.time_sec for m in meas]
    assert all(t > 0 for t in ts) and ts[-1] > ts[0], ts
    model = gs.fit_model(meas)
    assert model.a > 0 and model.b > 0
    comm.close()


@pytest.mark.parametrize("P", [2, 4])
def test_copy_engine_bf16_bit_exact(P):
    """bf16 gradients: the copies move bf16 bytes, the reduce widens to fp32,
    sums in rank order, rounds once to bf16 and applies it to the fp32
    master weights — the bf16 oracle's semantics."""
    rng = np.random.default_rng(950 + P)
    counts = RAGGED
    g_np = [[pyoracle.f32_to_bf16(rng.uniform(-1, 1, c).astype(np.float32)) for c in counts] for _ in range(P)]
    w_np = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    offs = [0]
    for c in counts:
        offs.append(offs[-1] + ((c + 7) & ~7))  # 16-byte aligned bf16 layers
    g_dev = []
    for per in g_np:
        b = torch.zeros(offs[-1], dtype=torch.bfloat16, device="cuda")
        for l, a in enumerate(per):
            b[offs[l]:offs[l] + counts[l]] = torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
        g_dev.append([b[offs[l]:offs[l] + counts[l]] for l in range(len(counts))])
    w_dev = [[torch.from_numpy(a.copy()).cuda() for a in per] for per in w_np]
    plan = gs.MergePlan.all_normal(len(counts))
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    assert dp.dtype == rt.BF16
    ce = rt.CopyEngine(dp, 0.01)
    s = torch.cuda.current_stream()
    for _ in range(2):
        ce.begin(s)
        for g in reversed(range(dp.n_groups)):
            ce.mark_ready(g, s)
        ce.join(s)
        pyoracle.allreduce_sgd_bf16(g_np, w_np, [int(t) for t in plan.tags], 0.01)
    torch.cuda.synchronize()
    ce.check()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    ce.close()
    dp.close()
    comm.close()
