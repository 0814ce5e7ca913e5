"""GPU parity of the sm_100a kernels against the CPU oracle (bit-exact) and,
at full size, against a plain torch fp32 rank-order reference.

Multi-rank collectives are exercised on ONE B200 through the loopback
communicator: P emulated ranks, every collective one cooperative launch
(never P launches that wait on each other). The multi-GPU path is
tests/test_gpu_multirank.py.
"""
import numpy as np
import pytest
import torch

from oracle import pyoracle
from paper_1912_09268_b200 import gradsched as gs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_09268_b200 import runtime as rt

RAGGED = [1000, 0, 7, 9000, 4096, 13, 20000, 1, 4097, 3]
LR = 0.01


def _np(rng, counts, P):
    return [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]


def _dev(arrays):
    return [[torch.from_numpy(a.copy()).cuda() for a in per] for per in arrays]


def _plan_for(counts, seed=1):
    rng = np.random.default_rng(seed)
    t_b = list(rng.uniform(1e-5, 5e-4, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 1e-3)
    return tr, gs.optimal_plan(tr, gs.AllReduceModel(3e-5, 1e-9))


def test_pack_kernel_bit_exact_incl_unaligned_views():
    rng = np.random.default_rng(11)
    counts = RAGGED
    g_np = _np(rng, counts, 1)[0]
    # layer 2 is an unaligned view (offset by one float) to force the scalar path
    base = torch.from_numpy(np.concatenate([[0.0], g_np[2]]).astype(np.float32)).cuda()
    g_dev = [torch.from_numpy(a).cuda() for a in g_np]
    g_dev[2] = base[1:]
    tr, plan = _plan_for(counts)
    comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev, None, plan)
    offs = pyoracle.merge_offsets(counts)
    for g, members in enumerate(plan.groups()):
        b, n, nbytes = dp.group_span(g)
        assert b == offs[members[0]] and n == offs[members[-1] + 1] - b
        assert nbytes == 4 * sum(counts[i] for i in members)
        out = torch.full((max(n, 1),), float("nan"), device="cuda")
        dp.pack(g, 0.25, out)
        torch.cuda.synchronize()
        want = pyoracle.pack(g_np, members[0], members[-1] + 1, 0.25)
        assert np.array_equal(out[:n].cpu().numpy(), want), g
    dp.close()
    comm.close()


def test_unpack_sgd_kernel_bit_exact():
    rng = np.random.default_rng(12)
    counts = RAGGED
    g_np = _np(rng, counts, 1)[0]
    w_np = _np(rng, counts, 1)[0]
    g_dev = [torch.from_numpy(a.copy()).cuda() for a in g_np]
    w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np]
    _, plan = _plan_for(counts)
    comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    for g, members in enumerate(plan.groups()):
        b, n, _ = dp.group_span(g)
        red_np = rng.uniform(-1, 1, max(n, 1)).astype(np.float32)
        dp.unpack_sgd(g, torch.from_numpy(red_np).cuda(), LR, write_grad=True)
        torch.cuda.synchronize()
        offs = pyoracle.merge_offsets(counts)
        for l in members:
            r = red_np[offs[l] - b: offs[l] - b + counts[l]]
            want_w = (w_np[l] - (np.float32(LR) * r).astype(np.float32)).astype(np.float32)
            assert np.array_equal(w_dev[l].cpu().numpy(), want_w), l
            assert np.array_equal(g_dev[l].cpu().numpy(), r), l
    dp.close()
    comm.close()


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot", "auto"])
@pytest.mark.parametrize("protocol", ["stream", "chunked"])
def test_fused_group_allreduce_bit_exact_vs_oracle(P, algo, protocol):
    if P == 1 and (algo != "auto" or protocol != "stream"):
        pytest.skip("P=1 has no exchange")
    rng = np.random.default_rng(100 + P)
    counts = RAGGED
    g_np, w_np = _np(rng, counts, P), _np(rng, counts, P)
    g_dev, w_dev = _dev(g_np), _dev(w_np)
    _, plan = _plan_for(counts, seed=P)
    tags = [int(t) for t in plan.tags]
    if P == 1:
        comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
        dp = rt.DevicePlan(comm, g_dev[0], w_dev[0], plan)
    else:
        comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
        comm.set_oneshot_max(16 * 1024)  # auto: small groups one-shot, big two-shot
        comm.set_protocol(protocol)
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    # three iterations (exercises the epoch counter and arena parity)
    for it in range(3):
        for g in reversed(range(dp.n_groups)):
            dp.group_allreduce(g, LR, rt.SGD | rt.WRITE_GRAD, algo)
        pyoracle.allreduce_sgd(g_np, w_np, tags, LR, write_grad=True)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
            assert np.array_equal(g_dev[r][l].cpu().numpy(), g_np[r][l]), (r, l)
    dp.close()
    comm.close()


@pytest.mark.parametrize("P,algo", [(8, "twoshot"), (8, "oneshot"), (4, "twoshot"), (2, "twoshot")])
def test_large_message_matches_torch_fp32_rank_order(P, algo):
    """64 MiB per rank, 3 layers: bit-exact against torch fp32 elementwise
    ops in rank order (separate mul/add kernels, no FMA)."""
    torch.manual_seed(P)
    counts = [16 * 1024 * 1024 - 5, 3, 1 << 20]
    grads = [[torch.rand(c, device="cuda") * 2 - 1 for c in counts] for _ in range(P)]
    weights = [[torch.rand(c, device="cuda") for c in counts] for _ in range(P)]
    s = torch.tensor(1.0 / P, device="cuda")
    lr = torch.tensor(LR, device="cuda")
    want_w = []
    for l in range(len(counts)):
        acc = grads[0][l] * s
        for r in range(1, P):
            acc = acc + grads[r][l] * s
        want_w.append([weights[r][l] - lr * acc for r in range(P)])
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    plan = gs.MergePlan.all_merged(len(counts))
    dp = rt.DevicePlan(comm, grads, weights, plan)
    dp.group_allreduce(0, LR, rt.SGD, algo)
    torch.cuda.synchronize()
    for l in range(len(counts)):
        for r in range(P):
            assert torch.equal(weights[r][l], want_w[l][r]), (l, r)
    dp.close()
    comm.close()


def test_zero_byte_group_is_a_noop_launch():
    counts = [100, 0, 0, 50]
    tags = [0, 0, 1, 0]  # group 1 = layers 1..2, zero bytes
    g = [[torch.ones(c, device="cuda") for c in counts] for _ in range(2)]
    w = [[torch.zeros(c, device="cuda") for c in counts] for _ in range(2)]
    comm = rt.Comm.create_loopback(2, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g, w, gs.MergePlan([gs.LayerTag(t) for t in tags]))
    assert dp.n_groups == 3 and dp.group_span(1)[2] == 0
    for gi in reversed(range(3)):
        dp.group_allreduce(gi, 1.0, rt.SGD)
    torch.cuda.synchronize()
    assert torch.all(w[0][0] == -1.0) and torch.all(w[1][3] == -1.0)
    dp.close()
    comm.close()


def test_plain_allreduce_p1_is_identity_and_calibration_fits():
    comm = rt.Comm(0, 1, 0, 64 << 20)
    x = torch.randn(1000003, device="cuda")
    y = x.clone()
    comm.allreduce_(y)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    sizes = [4096 << k for k in range(0, 13, 2)]
    model, meas = rt.calibrated_model(comm, sizes, warmup=2, reps=5)
    assert all(m.time_sec > 0 for m in meas)
    assert meas[-1].time_sec > meas[0].time_sec
    assert model.a > 0 and model.b >= 0
    meas_e = comm.calibrate_engine(sizes, warmup=1, reps=3)
    assert all(m.time_sec > 0 for m in meas_e)
    assert meas_e[-1].time_sec > meas_e[0].time_sec
    em = gs.fit_model(meas_e)
    assert em.a > 0 and em.b >= 0
    comm.close()


@pytest.mark.parametrize("engine_ctas", [0, -1, 8])
def test_pipeline_p1_replays_backward_and_applies_sgd(engine_ctas):
    rng = np.random.default_rng(5)
    counts = RAGGED
    t_b = list(rng.uniform(5e-5, 3e-4, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 2e-3)
    plan = gs.optimal_plan(tr, gs.AllReduceModel(5e-6, 1 / 3e12))
    g_np, w_np = _np(rng, counts, 1), _np(rng, counts, 1)
    g_dev, w_dev = _dev(g_np), _dev(w_np)
    comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev[0], w_dev[0], plan)
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=True, l2_flush_bytes=64 << 20,
                       engine_ctas=engine_ctas)
    ms = pipe.run(4)
    compute_ms = (tr.forward_time + sum(t_b)) * 1e3
    assert all(m >= compute_ms * 0.999 for m in ms), (ms, compute_ms)
    assert all(m < compute_ms + 2.0 for m in ms), (ms, compute_ms)
    gt = pipe.group_times_ms()
    assert len(gt) == dp.n_groups
    for g, members in enumerate(plan.groups()):  # zero-byte groups are no-ops in the engine
        assert gt[g] > 0 or (engine_ctas != 0 and sum(counts[i] for i in members) == 0), (g, gt)
    if engine_ctas != 0:
        tl = pipe.device_timeline()
        assert abs(tl["replay_us"] - compute_ms * 1e3) < 50.0, tl
        assert 0.0 <= tl["tail_us"] < 100.0, tl
    for _ in range(4):
        pyoracle.allreduce_sgd(g_np, w_np, [int(t) for t in plan.tags], LR)
    for l in range(len(counts)):
        assert np.array_equal(w_dev[0][l].cpu().numpy(), w_np[0][l]), l
    pipe.close()
    dp.close()
    comm.close()


def test_pipeline_step_io_copies_inputs_and_results():
    """mgw_pipeline_create_io: the step's gradients arrive H2D inside the
    graph (before any group kernel) and a result is read back D2H."""
    counts = [1000, 7, 50000]
    tr = gs.trace_from_arrays(counts, [1e-4, 1e-4, 2e-4], 5e-4)
    plan = gs.MergePlan.all_normal(3)
    flat = torch.zeros(rt.padded_elems(counts), device="cuda")
    offs = pyoracle.merge_offsets(counts)
    grads = [flat[offs[i]:offs[i] + c] for i, c in enumerate(counts)]
    weights = [torch.zeros(c, device="cuda") for c in counts]
    host_in = torch.ones(flat.numel(), pin_memory=True)
    host_out = torch.zeros(4, pin_memory=True)
    comm = rt.Comm(0, 1, 0, 4 * flat.numel())
    dp = rt.DevicePlan(comm, grads, weights, plan)
    for engine in (-1, 0):
        pipe = rt.Pipeline(dp, tr, 0.5, engine_ctas=engine, h2d=(host_in, flat), d2h=(host_out, weights[0][:4]))
        pipe.run(2)
        torch.cuda.synchronize()
        want = -1.0 if engine == -1 else -2.0  # two steps per pipeline, cumulative
        assert torch.all(weights[2] == want) and torch.all(host_out == want), (engine, host_out)
        pipe.close()
    dp.close()
    comm.close()


# ---- bf16 gradients: bit-exact vs the bf16 oracle ----------

def _bf16_np(rng, counts, P):
    return [[pyoracle.f32_to_bf16(rng.uniform(-1, 1, c).astype(np.float32)) for c in counts] for _ in range(P)]


def _bf16_dev(arrays):
    return [[torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16) for a in per] for per in arrays]


def _bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot", "auto"])
def test_bf16_fused_group_allreduce_bit_exact_vs_oracle(P, algo):
    if P == 1 and algo != "auto":
        pytest.skip("P=1 has no exchange")
    rng = np.random.default_rng(300 + P)
    counts = RAGGED
    g_np, w_np = _bf16_np(rng, counts, P), _np(rng, counts, P)
    g_dev, w_dev = _bf16_dev(g_np), _dev(w_np)
    _, plan = _plan_for(counts, seed=P)
    tags = [int(t) for t in plan.tags]
    if P == 1:
        comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
        dp = rt.DevicePlan(comm, g_dev[0], w_dev[0], plan)
    else:
        comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
        comm.set_oneshot_max(8 * 1024)
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    assert dp.dtype == rt.BF16
    for it in range(3):
        for g in reversed(range(dp.n_groups)):
            dp.group_allreduce(g, LR, rt.SGD | rt.WRITE_GRAD, algo)
        pyoracle.allreduce_sgd_bf16(g_np, w_np, tags, LR, write_grad=True)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(_bits(g_dev[r][l]), g_np[r][l]), (r, l)
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    dp.close()
    comm.close()


def test_bf16_pack_unpack_bit_exact():
    rng = np.random.default_rng(21)
    counts = RAGGED
    g_np = _bf16_np(rng, counts, 1)[0]
    w_np = _np(rng, counts, 1)[0]
    g_dev = _bf16_dev([g_np])[0]
    w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np]
    _, plan = _plan_for(counts)
    comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    offs = pyoracle.merge_offsets_granule(counts, 8)
    for g, members in enumerate(plan.groups()):
        b, n, nbytes = dp.group_span(g)
        assert b == offs[members[0]] and n == offs[members[-1] + 1] - b and nbytes == 2 * sum(counts[i] for i in members)
        out = torch.zeros(max(n, 1), dtype=torch.bfloat16, device="cuda")
        dp.pack(g, 0.5, out)
        torch.cuda.synchronize()
        want = pyoracle.pack_bf16(g_np, members[0], members[-1] + 1, 0.5)
        got = _bits(out)[:n]
        for l in members:  # compare the valid elements of every layer (padding is unspecified)
            o = offs[l] - b
            assert np.array_equal(got[o:o + counts[l]], want[o:o + counts[l]]), l
        red = pyoracle.f32_to_bf16(rng.uniform(-1, 1, max(n, 1)).astype(np.float32))
        red_dev = torch.from_numpy(red.view(np.int16).copy()).cuda().view(torch.bfloat16)
        w_before = [w_dev[l].cpu().numpy().copy() for l in members]
        dp.unpack_sgd(g, red_dev, LR, write_grad=True)
        torch.cuda.synchronize()
        for k, l in enumerate(members):
            r = pyoracle.bf16_to_f32(red[offs[l] - b: offs[l] - b + counts[l]])
            assert np.array_equal(w_dev[l].cpu().numpy(), (w_before[k] - (np.float32(LR) * r).astype(np.float32))), l
            assert np.array_equal(_bits(g_dev[l]), red[offs[l] - b: offs[l] - b + counts[l]]), l
    dp.close()
    comm.close()


@pytest.mark.parametrize("P,algo", [(4, "twoshot"), (2, "oneshot")])
def test_bf16_large_message_matches_torch_rank_order(P, algo):
    """32 Mi bf16 elements per rank: bit-exact against torch (fp32 widening,
    rank-order fp32 sum, one bf16 rounding, fp32 SGD)."""
    torch.manual_seed(10 + P)
    counts = [32 * 1024 * 1024 - 3, 5, 1 << 20]
    grads = [[(torch.rand(c, device="cuda") * 2 - 1).to(torch.bfloat16) for c in counts] for _ in range(P)]
    weights = [[torch.rand(c, device="cuda") for c in counts] for _ in range(P)]
    s = torch.tensor(1.0 / P, device="cuda")
    lr = torch.tensor(LR, device="cuda")
    want_w, want_g = [], []
    for l in range(len(counts)):
        acc = grads[0][l].float() * s
        for r in range(1, P):
            acc = acc + grads[r][l].float() * s
        red = acc.to(torch.bfloat16)
        want_g.append(red)
        want_w.append([weights[r][l] - lr * red.float() for r in range(P)])
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts, rt.BF16))
    dp = rt.DevicePlan(comm, grads, weights, gs.MergePlan.all_merged(len(counts)))
    dp.group_allreduce(0, LR, rt.SGD | rt.WRITE_GRAD, algo)
    torch.cuda.synchronize()
    for l in range(len(counts)):
        for r in range(P):
            assert torch.equal(weights[r][l], want_w[l][r]), (l, r)
            assert torch.equal(grads[r][l], want_g[l]), (l, r)
    dp.close()
    comm.close()
