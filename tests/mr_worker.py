"""Multi-GPU parity worker (launched by tests/test_gpu_multirank.py through
torch.distributed.run, one process per GPU, NCCL for the plumbing).

Every rank builds seeded gradients/weights, maps the peers' merge arenas
over NVLink (CUDA IPC), runs the fused per-group all-reduce (one-shot,
two-shot, auto) for several iterations, and checks the result bit-for-bit
against the CPU oracle fed with ALL ranks' inputs (regenerated locally from
the seeds). Also: plain SUM all-reduce vs NCCL (norm-wise bound), a pipeline
run, and a calibration sweep whose fit must be usable by the planner.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from paper_1912_09268_b200 import dist as D  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

COUNTS = [1000, 0, 7, 9000, 4096, 13, 200000, 1, 4097, 3, 3_000_000]
LR = 0.01


def inputs(P):
    g = [[np.random.default_rng(0x5EED0000 + r).uniform(-1, 1, c).astype(np.float32) for c in COUNTS]
         for r in range(P)]
    w = [[np.random.default_rng(0xC0FFEE).uniform(-1, 1, c).astype(np.float32) for c in COUNTS]
         for _ in range(P)]
    return g, w


def group_oracle(g_np, w_np, tags, thr, write_grad):
    """One iteration of the oracle, group by group: NVLS numerics for fp32
    groups of >= thr bytes (thr 0: every group), rank order otherwise."""
    heads = [i for i, t in enumerate(tags) if i == 0 or t == 0] + [len(tags)]
    for a, b in zip(heads, heads[1:]):
        nbytes = 4 * sum(COUNTS[a:b])
        fn = pyoracle.allreduce_sgd_nvls if (thr == 0 or nbytes >= thr) else pyoracle.allreduce_sgd
        gs_ = [per[a:b] for per in g_np]
        ws_ = [per[a:b] for per in w_np]
        fn(gs_, ws_, [0] + [1] * (b - a - 1), LR, write_grad=write_grad)


def nvls_checks(comm, plan, tags, tr, rank, P):
    failures = []
    for algo, thr in (("nvls", 0), ("auto", 1 << 20)):
        comm.set_nvls(thr if algo == "auto" else 0, 2)
        g_np, w_np = inputs(P)
        g_dev = [torch.from_numpy(a.copy()).cuda() for a in g_np[rank]]
        w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np[rank]]
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
        for _ in range(3):
            for g in reversed(range(dp.n_groups)):
                dp.group_allreduce(g, LR, rt.SGD | rt.WRITE_GRAD, algo)
            group_oracle(g_np, w_np, tags, thr, True)
        torch.cuda.synchronize()
        for l in range(len(COUNTS)):
            if not np.array_equal(w_dev[l].cpu().numpy(), w_np[rank][l]):
                failures.append(f"nvls {algo} weights layer {l}")
            if not np.array_equal(g_dev[l].cpu().numpy(), g_np[rank][l]):
                failures.append(f"nvls {algo} grads layer {l}")
        dp.close()
    # pipeline: engine (AUTO protocol: streamed) + the last-ready group as a
    # standalone launch, NVLS when it is >= 1 MiB
    comm.set_nvls(1 << 20, 2)
    g_np, w_np = inputs(P)
    g_dev = [torch.from_numpy(a.copy()).cuda() for a in g_np[rank]]
    w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np[rank]]
    dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
    pipe = rt.Pipeline(dp, tr, LR, record_group_times=True, l2_flush_bytes=0, engine_ctas=-1)
    pipe.run(3)
    torch.cuda.synchronize()
    heads = [i for i, t in enumerate(tags) if i == 0 or t == 0] + [len(tags)]
    tail_bytes = 4 * sum(COUNTS[heads[0]:heads[1]])
    for _ in range(3):  # the engine's groups [1, G) are push groups; group 0 is the tail launch
        for a, b in zip(heads, heads[1:]):
            fn = pyoracle.allreduce_sgd_nvls if (a == 0 and tail_bytes >= (1 << 20)) else pyoracle.allreduce_sgd
            fn([per[a:b] for per in g_np], [per[a:b] for per in w_np], [0] + [1] * (b - a - 1), LR)
    for l in range(len(COUNTS)):
        if not np.array_equal(w_dev[l].cpu().numpy(), w_np[rank][l]):
            failures.append(f"nvls pipeline weights layer {l}")
    pipe.close()
    dp.close()
    # plain SUM all-reduce through the switch vs NCCL (norm-wise bound)
    for n in (1 << 10, (1 << 20) + 3, 16 << 20):
        x = torch.rand(n, device="cuda") * 2 - 1 + rank
        mine, ref = x.clone(), x.clone()
        comm.allreduce_(mine, algo="nvls")
        dist.all_reduce(ref)
        absx = x.abs()
        dist.all_reduce(absx)
        torch.cuda.synchronize()
        if not bool(((mine - ref).abs() <= 1e-6 * absx + 1e-30).all()):
            failures.append(f"nvls allreduce vs nccl n={n}")
    meas = comm.calibrate([1 << 20, 16 << 20, 64 << 20], warmup=2, reps=5, algo="nvls")
    if rank == 0:
        print("nvls calibration", [(m.size_bytes, round(m.time_sec * 1e6, 1)) for m in meas], flush=True)
    return failures


def main():
    rank, P, local = D.init("nccl")
    torch.cuda.set_device(local)
    rng = np.random.default_rng(9)
    t_b = list(rng.uniform(1e-5, 4e-4, len(COUNTS)))
    tr = gs.trace_from_arrays(COUNTS, t_b, 1e-3)
    plan = gs.optimal_plan(tr, gs.AllReduceModel(2e-5, 1 / 500e9))
    D.agree_plan(plan.tags)
    tags = [int(t) for t in plan.tags]
    comm = rt.Comm(rank, P, local, max(4 * rt.padded_elems(COUNTS), 80 << 20))
    assert comm.num_peers() == P, comm.num_peers()
    comm.set_oneshot_max(64 * 1024)
    failures = []
    for algo in ("oneshot", "twoshot", "auto"):
        g_np, w_np = inputs(P)
        g_dev = [torch.from_numpy(a.copy()).cuda() for a in g_np[rank]]
        w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np[rank]]
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
        for _ in range(3):
            for g in reversed(range(dp.n_groups)):
                dp.group_allreduce(g, LR, rt.SGD | rt.WRITE_GRAD, algo)
            pyoracle.allreduce_sgd(g_np, w_np, tags, LR, write_grad=True)
        torch.cuda.synchronize()
        for l in range(len(COUNTS)):
            if not np.array_equal(w_dev[l].cpu().numpy(), w_np[rank][l]):
                failures.append(f"{algo} weights layer {l}")
            if not np.array_equal(g_dev[l].cpu().numpy(), g_np[rank][l]):
                failures.append(f"{algo} grads layer {l}")
        dp.close()

    # bf16 gradients (fp32 master weights) over real NVLink: bit-exact vs the
    # bf16 oracle, every algorithm
    for algo in ("oneshot", "twoshot", "auto"):
        g32, w_np = inputs(P)
        g_np = [[pyoracle.f32_to_bf16(a) for a in per] for per in g32]
        g_dev = [torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16) for a in g_np[rank]]
        w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np[rank]]
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
        for _ in range(2):
            for g in reversed(range(dp.n_groups)):
                dp.group_allreduce(g, LR, rt.SGD | rt.WRITE_GRAD, algo)
            pyoracle.allreduce_sgd_bf16(g_np, w_np, tags, LR, write_grad=True)
        torch.cuda.synchronize()
        for l in range(len(COUNTS)):
            if not np.array_equal(w_dev[l].cpu().numpy(), w_np[rank][l]):
                failures.append(f"bf16 {algo} weights layer {l}")
            if not np.array_equal(g_dev[l].view(torch.int16).cpu().numpy().view(np.uint16), g_np[rank][l]):
                failures.append(f"bf16 {algo} grads layer {l}")
        dp.close()

    # plain SUM all-reduce vs NCCL: bit-exact is not expected (NCCL's order
    # differs); bound |x - y| <= 1e-6 * sum_r |x_r| (SURVEY §7 vii)
    for n in (1 << 10, (1 << 20) + 3, 16 << 20):
        x = torch.rand(n, device="cuda") * 2 - 1 + rank
        mine, ref = x.clone(), x.clone()
        comm.allreduce_(mine)
        dist.all_reduce(ref)
        absx = x.abs()
        dist.all_reduce(absx)
        torch.cuda.synchronize()
        if not bool(((mine - ref).abs() <= 1e-6 * absx + 1e-30).all()):
            failures.append(f"allreduce vs nccl n={n}")

    # pipelines at P ranks (per-group launches and the persistent engine):
    # 5 iterations of SGD with the static gradients, bit-exact vs the oracle
    for engine in (0, -1, 16):
        g_np, w_np = inputs(P)
        g_dev = [torch.from_numpy(a.copy()).cuda() for a in g_np[rank]]
        w_dev = [torch.from_numpy(a.copy()).cuda() for a in w_np[rank]]
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
        pipe = rt.Pipeline(dp, tr, LR, record_group_times=True, l2_flush_bytes=64 << 20, engine_ctas=engine)
        ms = pipe.run(5)
        gt = pipe.group_times_ms()
        compute_ms = (tr.forward_time + sum(t_b)) * 1e3
        if not all(m >= compute_ms * 0.999 for m in ms):
            failures.append(f"engine={engine}: pipeline faster than its compute: {ms} < {compute_ms}")
        if not all(t >= 0 for t in gt) or sum(gt) <= 0:
            failures.append(f"engine={engine}: bad group times {gt}")
        for _ in range(5):
            pyoracle.allreduce_sgd(g_np, w_np, tags, LR)
        for l in range(len(COUNTS)):
            if not np.array_equal(w_dev[l].cpu().numpy(), w_np[rank][l]):
                failures.append(f"engine={engine}: pipeline weights layer {l}")
        pipe.close()
        dp.close()

    # real backward (autograd hooks -> engine), each rank on different data:
    # weights after the step == W - lr * (g_0/P + ... + g_{P-1}/P), rank order
    from paper_1912_09268_b200.ddp import MGWFBP

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 10)).cuda()
    L = len(list(model.parameters()))
    mplan = gs.MergePlan([gs.LayerTag(0 if i % 2 == 0 else 1) for i in range(L)])
    gen = torch.Generator(device="cuda").manual_seed(100 + rank)
    for step in range(9):
        if step % 3 == 0:  # steps 0-2: persistent engine; 3-5: one launch per group; 6-8: copy engines
            if step:
                sync.check()
                sync.close()
            sync = MGWFBP(model, comm, LR, plan=mplan, engine_ctas=8, mode=("engine", "launch", "ce")[step // 3],
                          launch_ctas=4)
        w_before = [p.detach().cpu().numpy().copy() for p in model.parameters()]
        x = torch.randn(16, 64, device="cuda", generator=gen)
        y = torch.randint(0, 10, (16,), device="cuda", generator=gen)
        sync.begin()
        torch.nn.functional.cross_entropy(model(x), y).backward()
        sync.end()
        torch.cuda.synchronize()
        grads = [None] * P
        dist.all_gather_object(grads, [p.grad.detach().cpu().numpy().copy() for p in model.parameters()])
        s = np.float32(1.0 / P)
        for li, p in enumerate(model.parameters()):
            acc = (grads[0][li] * s).astype(np.float32)
            for r in range(1, P):
                acc = (acc + (grads[r][li] * s).astype(np.float32)).astype(np.float32)
            want = (w_before[li] - (np.float32(LR) * acc).astype(np.float32)).astype(np.float32)
            if not np.array_equal(p.detach().cpu().numpy(), want):
                failures.append(f"real backward step {step} param {li}")
    sync.check()
    sync.close()

    # memory-ordering stress over real NVLink: 30 engine iterations with NEW
    # gradients every iteration (every rank regenerates all ranks' gradients
    # from the shared seeds), both protocols, bit-exact vs torch fp32
    # rank-order ops after every iteration
    for protocol in ("chunked", "stream"):
        comm.set_protocol(protocol)
        gens = [torch.Generator(device="cuda").manual_seed(500 + r) for r in range(P)]
        wgen = torch.Generator(device="cuda").manual_seed(499)
        g_all = [[torch.empty(c, device="cuda") for c in COUNTS] for _ in range(P)]
        w_dev = [torch.empty(c, device="cuda").uniform_(-1, 1, generator=wgen) for c in COUNTS]
        want = [w.clone() for w in w_dev]
        g_dev = [torch.empty(c, device="cuda") for c in COUNTS]
        dp = rt.DevicePlan(comm, g_dev, w_dev, plan)
        pipe = rt.Pipeline(dp, tr, LR, record_group_times=False, l2_flush_bytes=0, engine_ctas=-1)
        sc = 1.0 / P
        for it in range(30):
            for r in range(P):
                for g in g_all[r]:
                    g.uniform_(-1, 1, generator=gens[r])
            for l in range(len(COUNTS)):
                g_dev[l].copy_(g_all[rank][l])
            torch.cuda.synchronize()
            pipe.run(1)
            torch.cuda.synchronize()
            for l in range(len(COUNTS)):
                red = g_all[0][l] * sc
                for r in range(1, P):
                    red = red + g_all[r][l] * sc
                want[l] = want[l] - LR * red
                if not torch.equal(w_dev[l], want[l]):
                    failures.append(f"stress {protocol} iteration {it} layer {l}")
                    want[l] = w_dev[l].clone()
        pipe.close()
        dp.close()
    comm.set_protocol("chunked")

    # NVLS (switch-reduced, opt-in): bit-exact vs the oracle's exact-sum
    # variant (== the rank-order oracle at P = 2). Every group forced through
    # NVLS; then AUTO with a 1 MiB threshold (mixed NVLS / push groups), the
    # pipeline (persistent engine + the tail group as a standalone NVLS
    # launch), and the plain SUM all-reduce vs NCCL.
    if comm.nvls_supported():
        comm.enable_nvls(min_bytes=0, chunk_tiles=2)
        failures += nvls_checks(comm, plan, tags, tr, rank, P)
        comm.set_nvls(0)
    else:
        print(f"rank {rank}: NVLS unsupported, skipped", flush=True)

    meas = comm.calibrate([4096 << k for k in range(0, 12, 2)], warmup=2, reps=5)  # <= arena
    meas_e = comm.calibrate_engine([4096 << k for k in range(0, 12, 2)], warmup=1, reps=3)
    for mm in (meas, meas_e):
        try:
            gs.fit_model(mm)
        except gs.FitError as e:
            failures.append(f"calibration fit: {e}")
    comm.close()
    out = [None] * P
    dist.all_gather_object(out, failures)
    if rank == 0:
        bad = [f for per in out for f in per]
        print("MULTIRANK", "OK" if not bad else "FAIL", bad, flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
