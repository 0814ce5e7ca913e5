"""The persistent comm engine at P > 1 on ONE B200 (loopback communicator:
P emulated ranks, one engine grid (ctas, P) per iteration).

This is the kernel every N > 1 bench row runs on: LL, one-shot and two-shot
groups mixed in one launch, FIFO in backward order (the serialised schedule
of reference timeline.hpp:133-154), groups rotated over the CTAs, the
backward replayed from the trace. Parity: bit-exact vs the CPU oracle
(oracle/mgw_oracle.c, rank-order fp32 sum, x 1/P per source, SGD with two
roundings) on the ragged and ResNet-50 traces; on BERT-large (336 M
parameters per rank) every layer is checked bit-exact against torch fp32
rank-order ops on the GPU and a sample of layers against the C oracle.
Plans come from the committed on-box calibrations (profiles/calib) through
the reference's fit_model + optimal_plan (planner.hpp:63-98).
"""
import os

import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import pyoracle
from paper_1912_09268_b200 import gradsched as gs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_09268_b200 import runtime as rt

RAGGED = [1000, 0, 7, 9000, 4096, 13, 20000, 1, 4097, 3, 300000, 5, 1 << 20, 77]
LR = 0.01


def _np(rng, counts, P):
    return [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]


def _dev(arrays):
    return [[torch.from_numpy(a.copy()).cuda() for a in per] for per in arrays]


def committed_model(trace_name: str, P: int) -> gs.AllReduceModel:
    """fit_model over the committed on-box calibration of this trace at P
    (the nearest measured P below when P has none)."""
    for q in (P, 4, 2):
        path = os.path.join(ROOT, "profiles", "calib", f"calib_{trace_name}_P{q}.csv")
        if q <= P and os.path.exists(path):
            return gs.fit_model(gs.load_measurements_csv(path))
    raise FileNotFoundError(trace_name)


def algo_mix(dp, comm):
    """(LL, one-shot, two-shot) group counts of a plan under the comm's thresholds."""
    ll = one = two = 0
    for g in range(dp.n_groups):
        nbytes = dp.group_span(g)[2]
        if nbytes == 0:
            continue
        if nbytes > comm.oneshot_max:
            two += 1
        elif nbytes <= comm.ll_max_bytes:
            ll += 1
        else:
            one += 1
    return ll, one, two


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("protocol", ["stream", "chunked", "auto"])
def test_engine_pipeline_ragged_bit_exact(P, protocol):
    """Replay pipeline, 3 iterations, LL + one-shot + two-shot groups in one
    engine launch; the rank-order result on every emulated rank. AUTO (the
    default) runs the chunked engine at P > 1; STREAM the streamed engine
    plus the last-ready group as a chunked launch after it."""
    rng = np.random.default_rng(700 + P)
    counts = RAGGED
    t_b = list(rng.uniform(2e-5, 2e-4, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 3e-4)
    plan = gs.optimal_plan(tr, gs.AllReduceModel(6e-6, 1 / 600e9))
    tags = [int(t) for t in plan.tags]
    g_np, w_np = _np(rng, counts, P), _np(rng, counts, P)
    g_dev, w_dev = _dev(g_np), _dev(w_np)
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    assert comm.num_peers() == P
    comm.set_oneshot_max(256 * 1024)
    comm.set_ll_max(16 * 1024)
    comm.set_protocol(protocol)
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=True, l2_flush_bytes=32 << 20, engine_ctas=-1)
    assert pipe.engine_protocol == ("stream" if protocol == "stream" else "chunked")
    ms = pipe.run(3)
    compute_ms = (tr.forward_time + sum(t_b)) * 1e3
    assert all(m >= compute_ms * 0.999 for m in ms), (ms, compute_ms)
    for _ in range(3):
        pyoracle.allreduce_sgd(g_np, w_np, tags, LR)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    gt = pipe.group_times_ms()
    assert all(t > 0 for g, t in enumerate(gt) if dp.group_span(g)[2] > 0), gt
    assert not comm.failed()
    pipe.close()
    dp.close()
    comm.close()


def test_engine_pipeline_resnet50_p2_bit_exact():
    """BASELINE config 1: the ResNet-50 trace (161 tensors, 25.6 M fp32),
    its optimal plan under the committed P = 2 calibration, 2 ranks, 3
    replayed iterations through the engine — bit-exact vs the C oracle."""
    P = 2
    tr = gs.load_trace(os.path.join(ROOT, "traces", "resnet50.json"))
    plan = gs.optimal_plan(tr, committed_model("resnet50", P))
    tags = [int(t) for t in plan.tags]
    counts = [l.params for l in tr.layers]
    rng = np.random.default_rng(0x5EED0000)
    g_np, w_np = _np(rng, counts, P), _np(rng, counts, P)
    g_dev, w_dev = _dev(g_np), _dev(w_np)
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    ll, one, two = algo_mix(dp, comm)
    assert ll > 0 and two > 0, (ll, one, two)  # several protocols in one engine launch
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=False, l2_flush_bytes=64 << 20, engine_ctas=-1)
    pipe.run(3)
    for _ in range(3):
        pyoracle.allreduce_sgd(g_np, w_np, tags, LR)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    assert not comm.failed()
    pipe.close()
    dp.close()
    comm.close()


@pytest.mark.parametrize("P", [4, 8])
def test_engine_pipeline_bert_large_full_size(P):
    """BASELINE config 5 at full size (398 tensors, 336 M fp32 params per
    rank, 1.35 GB): optimal plan under the committed calibration, 3 replayed
    iterations through the loopback engine. Every layer bit-exact vs torch
    fp32 rank-order ops (separate mul / add / sub kernels: no FMA); every
    20th layer and the largest bit-exact vs the C oracle."""
    tr = gs.load_trace(os.path.join(ROOT, "traces", "bert_large.json"))
    plan = gs.optimal_plan(tr, committed_model("bert_large", P))
    counts = [l.params for l in tr.layers]
    L = len(counts)
    torch.cuda.empty_cache()
    gen = torch.Generator(device="cuda")
    grads, weights = [], []
    for r in range(P):
        gen.manual_seed(0x5EED0000 + r)
        grads.append([torch.empty(c, device="cuda").uniform_(-1, 1, generator=gen) for c in counts])
        gen.manual_seed(0xC0FFEE + r)
        weights.append([torch.empty(c, device="cuda").uniform_(-1, 1, generator=gen) for c in counts])
    sample = sorted(set(range(0, L, 20)) | {int(np.argmax(counts))})
    g_np = [[grads[r][l].cpu().numpy() for l in sample] for r in range(P)]
    w_np = [[weights[r][l].cpu().numpy() for l in sample] for r in range(P)]
    want = [[w.clone() for w in per] for per in weights]
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, grads, weights, plan)
    ll, one, two = algo_mix(dp, comm)
    assert two > 0 and (ll + one) > 0, (ll, one, two)
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=False, l2_flush_bytes=0, engine_ctas=-1)
    pipe.run(3)
    torch.cuda.synchronize()
    assert not comm.failed()
    s = torch.tensor(1.0 / P, device="cuda")
    lr = torch.tensor(LR, device="cuda")
    for l in range(L):
        acc = grads[0][l] * s
        for r in range(1, P):
            acc = acc + grads[r][l] * s
        step = lr * acc
        for r in range(P):
            for _ in range(3):
                want[r][l] = want[r][l] - step
            assert torch.equal(weights[r][l], want[r][l]), (l, r)
        del acc, step
    for _ in range(3):
        pyoracle.allreduce_sgd(g_np, w_np, [0] * len(sample), LR)
    for r in range(P):
        for k, l in enumerate(sample):
            assert np.array_equal(weights[r][l].cpu().numpy(), w_np[r][k]), (r, l)
    pipe.close()
    dp.close()
    comm.close()
    del grads, weights, want
    torch.cuda.empty_cache()


def test_ll_epochs_unique_across_plans_on_one_comm():
    """LL packets of an earlier launch must never satisfy a later
    one. Two plans with different LL layouts (every layer its own LL group
    vs merged groups) and different CTA mappings (engine vs standalone
    launches, different grids) alternate on ONE communicator; the epoch is
    the communicator's launch sequence, unique per launch."""
    P = 2
    rng = np.random.default_rng(41)
    counts = [3000, 17, 5000, 64, 1200, 9, 4096, 333]
    t_b = list(rng.uniform(1e-5, 5e-5, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 1e-4)
    plans = [gs.MergePlan.all_normal(len(counts)),
             gs.MergePlan([gs.LayerTag(t) for t in [0, 1, 0, 1, 1, 0, 1, 1]])]
    g_np, w_np = _np(rng, counts, P), _np(rng, counts, P)
    g_dev, w_dev = _dev(g_np), _dev(w_np)
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    dps = [rt.DevicePlan(comm, g_dev, w_dev, p) for p in plans]
    pipes = [rt.Pipeline(dp, tr, LR, engine_ctas=c) for dp, c in zip(dps, (-1, 5))]
    for it in range(6):
        k = it % 2
        if it % 3 == 2:  # standalone launches of the same plan in between
            for g in reversed(range(dps[k].n_groups)):
                dps[k].group_allreduce(g, LR, rt.SGD)
        else:
            pipes[k].run(1)
        pyoracle.allreduce_sgd(g_np, w_np, [int(t) for t in plans[k].tags], LR)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    assert not comm.failed()
    for p in pipes:
        p.close()
    for dp in dps:
        dp.close()
    comm.close()


@pytest.mark.parametrize("P", [1, 2, 4])
def test_engine_drain_streams_whole_plan_bit_exact(P):
    """The standalone drain (every group ready at launch: the roofline / ncu
    kernel) applies exactly one SGD step per launch."""
    rng = np.random.default_rng(800 + P)
    counts = RAGGED
    t_b = list(rng.uniform(2e-5, 2e-4, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 3e-4)
    plan = gs.optimal_plan(tr, gs.AllReduceModel(4e-6, 1 / 900e9))
    tags = [int(t) for t in plan.tags]
    g_np, w_np = _np(rng, counts, P), _np(rng, counts, P)
    g_dev, w_dev = _dev(g_np), _dev(w_np)
    if P == 1:
        comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
        dp = rt.DevicePlan(comm, g_dev[0], w_dev[0], plan)
    else:
        comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
        comm.set_oneshot_max(64 * 1024)
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=True, l2_flush_bytes=32 << 20, engine_ctas=-1)
    ms = pipe.drain(2)
    assert len(ms) == 2 and all(m > 0 for m in ms)
    pipe.run(1)  # a replayed iteration after the drains (iteration counter stays consistent)
    for _ in range(3):
        pyoracle.allreduce_sgd(g_np, w_np, tags, LR)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    pipe.close()
    dp.close()
    comm.close()


def test_ready_timeout_fails_loudly_and_skips_sgd():
    """A group that is never marked ready: the engine gives up after its
    10 s bound, raises the communicator's host-mapped error flag, skips the
    SGD of every group it could not run, and mgw_engine_check reports it."""
    import ctypes as C

    from paper_1912_09268_b200 import _lib

    counts = [4096, 4096]
    g = [[torch.ones(c, device="cuda") for c in counts] for _ in range(2)]
    w = [[torch.zeros(c, device="cuda") for c in counts] for _ in range(2)]
    comm = rt.Comm.create_loopback(2, 0, 4 * rt.padded_elems(counts))
    dp = rt.DevicePlan(comm, g, w, gs.MergePlan.all_normal(2))
    h = C.c_void_p()
    gs.check(_lib.mgw_engine_create(dp.handle, 1.0, 0, 4, 0, C.byref(h)))
    s = torch.cuda.Stream()
    gs.check(_lib.mgw_engine_begin(h, s.cuda_stream))
    gs.check(_lib.mgw_engine_mark_ready(h, 1, s.cuda_stream))  # group 0 never
    assert _lib.mgw_engine_check(h) != 0
    assert b"timed out" in _lib.mgw_last_error()
    assert comm.failed()
    assert torch.all(w[0][1] == -1.0) and torch.all(w[1][1] == -1.0)  # group 1 ran
    assert torch.all(w[0][0] == 0.0) and torch.all(w[1][0] == 0.0)  # group 0: no SGD
    gs.check(_lib.mgw_pipeline_destroy(h))
    dp.close()
    comm.close()


@pytest.mark.parametrize("P,protocol", [(2, "chunked"), (2, "stream"), (4, "chunked"), (4, "stream"),
                                        (8, "stream")])
def test_ordering_stress_fresh_gradients_every_iteration(P, protocol):
    """Memory-ordering stress (compute-sanitizer is closed on this pool): 60
    engine iterations, NEW gradients every iteration (so a reduction that
    read a stale arena slot, LL packet or peer push would show), a plan
    mixing LL, one-shot and two-shot groups; after every iteration the
    weights must equal torch fp32 rank-order ops on the GPU bit for bit:
    w -= lr * (g_0 * s + g_1 * s + ...), separate rounded mul / add kernels."""
    rng = np.random.default_rng(1234 + P)
    counts = [700, 9000, 13, 70000, 4096, 1, 300000, 77, 2 << 20, 5000]
    t_b = list(rng.uniform(1e-5, 6e-5, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 1e-4)
    plan = gs.optimal_plan(tr, gs.AllReduceModel(5e-6, 1 / 600e9))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(77 + P)
    g_dev = [[torch.empty(c, device="cuda") for c in counts] for _ in range(P)]
    w0 = [torch.empty(c, device="cuda").uniform_(-1, 1, generator=gen) for c in counts]
    w_dev = [[w.clone() for w in w0] for _ in range(P)]  # data parallel: identical weights on every rank
    want = [w.clone() for w in w0]
    comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
    comm.set_oneshot_max(256 * 1024)
    comm.set_ll_max(32 * 1024)
    comm.set_protocol(protocol)
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    ll, one, two = algo_mix(dp, comm)
    assert ll > 0 and one > 0 and two > 0, (ll, one, two)
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=False, l2_flush_bytes=0, engine_ctas=-1)
    s = 1.0 / P
    for it in range(60):
        for r in range(P):
            for g in g_dev[r]:
                g.uniform_(-1, 1, generator=gen)
        torch.cuda.synchronize()  # the pipeline runs on its own streams
        pipe.run(1)
        torch.cuda.synchronize()
        for l in range(len(counts)):
            red = g_dev[0][l] * s
            for r in range(1, P):
                red = red + g_dev[r][l] * s
            want[l] = want[l] - LR * red
        for r in range(P):
            for l in range(len(counts)):
                assert torch.equal(w_dev[r][l], want[l]), (it, r, l)
    assert not comm.failed()
    pipe.close()
    dp.close()
    comm.close()


@pytest.mark.parametrize("P,protocol", [(1, "stream"), (1, "chunked"), (2, "chunked"), (2, "stream"),
                                        (4, "chunked"), (4, "stream")])
def test_engine_pipeline_bf16_bit_exact(P, protocol):
    """bf16 gradients through the persistent engine (P = 1: the TMA-fed
    single-rank engine — `stream` — and the register engine — `chunked`),
    3 replayed iterations, vs the bf16 oracle (fp32 rank-order sum, one
    rounding to bf16, fp32 master weights)."""
    rng = np.random.default_rng(1500 + P)
    counts = RAGGED
    t_b = list(rng.uniform(2e-5, 2e-4, len(counts)))
    tr = gs.trace_from_arrays(counts, t_b, 3e-4)
    tr.bytes_per_element = 2
    plan = gs.optimal_plan(tr, gs.AllReduceModel(6e-6, 1 / 600e9))
    tags = [int(t) for t in plan.tags]
    g_np = [[pyoracle.f32_to_bf16(rng.uniform(-1, 1, c).astype(np.float32)) for c in counts] for _ in range(P)]
    w_np = _np(rng, counts, P)
    g_dev = [[torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16) for a in per] for per in g_np]
    w_dev = _dev(w_np)
    if P == 1:
        comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
        comm.set_protocol(protocol)
        dp = rt.DevicePlan(comm, g_dev[0], w_dev[0], plan)
    else:
        comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
        comm.set_oneshot_max(256 * 1024)
        comm.set_ll_max(16 * 1024)
        comm.set_protocol(protocol)
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    assert dp.dtype == rt.BF16
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=False, l2_flush_bytes=32 << 20, engine_ctas=-1)
    pipe.run(3)
    for _ in range(3):
        pyoracle.allreduce_sgd_bf16(g_np, w_np, tags, LR)
    torch.cuda.synchronize()
    for r in range(P):
        for l in range(len(counts)):
            assert np.array_equal(w_dev[r][l].cpu().numpy(), w_np[r][l]), (r, l)
    assert not comm.failed()
    pipe.close()
    dp.close()
    comm.close()
