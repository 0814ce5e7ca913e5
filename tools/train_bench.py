"""Real-training comparison (paper §6 "real experiments"):
a torchvision model (or BERT-large pre-training) trained with synthetic data on N GPUs (torchrun, one
process per GPU), gradients synchronised by
  ddp        torch DistributedDataParallel (NCCL, 25 MB buckets) + torch SGD
  mgwfbp     this repo's persistent comm engine, optimal merge plan from the
             model's B200-measured trace + the on-box calibration
  wfbp       same engine, every layer its own group
  single     same engine, one group (single buffer)
Prints one JSON line per strategy (rank 0): median iteration ms, images/s.

usage: torchrun --nproc-per-node N tools/train_bench.py --model resnet50 --batch 32
"""
from __future__ import annotations

import argparse
import time
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1912_09268_b200 import dist as D  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402
from paper_1912_09268_b200.ddp import MGWFBP  # noqa: E402


sys.path.insert(0, os.path.join(ROOT, "tools"))
from extract_traces import build, loss_of, make_batch  # noqa: E402  (same models / inputs as the traces)


def time_loop(step, iters, warmup):
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    D.barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
    evs[0].record()
    host = []
    for i in range(iters):
        t0 = time.perf_counter()
        step()
        host.append((time.perf_counter() - t0) * 1e3)
        evs[i + 1].record()
    torch.cuda.synchronize()
    ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(iters)]
    time_loop.host_ms = statistics.median(host)  # host time to enqueue one step (no sync)
    return D.max_over_ranks(statistics.median(ms))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--engine-ctas", type=int, default=8)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--strategies", default="ddp,mgwfbp,wfbp,single")
    ap.add_argument("--tail-groups", type=int, default=1)
    ap.add_argument("--mode", default="engine", choices=["engine", "launch", "ce"],
                    help="mgwfbp / wfbp: persistent engine, per-group launches, or copy-engine pushes + one "
                         "reduce after the backward (single always: one full-width launch after the backward)")
    ap.add_argument("--launch-ctas", type=int, default=16)
    ap.add_argument("--debug", action="store_true")
    args = ap.parse_args()
    rank, N, local = D.init("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.backends.cudnn.benchmark = True
    batch = make_batch(args.model, args.batch, dev)
    trace = gs.load_trace(os.path.join(ROOT, "traces", f"{args.model}.json"))
    results = {}

    phase_ev = []  # (after forward, after backward) event pairs of the timed steps

    def fwd_bwd(model):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_of(args.model, model, batch)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        loss.backward()
        e[1].record()
        phase_ev.append(e)

    for strat in args.strategies.split(","):
        torch.manual_seed(0)
        model = build(args.model).to(dev).train()
        if strat == "ddp":
            if N > 1:
                ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], bucket_cap_mb=25)
            else:
                ddp = model
            opt = torch.optim.SGD(model.parameters(), lr=args.lr)

            def step():
                opt.zero_grad(set_to_none=False)
                fwd_bwd(ddp)
                opt.step()

            ms = time_loop(step, args.iters, args.warmup)
            results[strat] = {"iter_ms": ms}
            del ddp, opt
        else:
            named = dict(model.named_parameters())
            params = [named[l.name] for l in trace.layers]  # the trace's layer order
            counts = [p.numel() for p in params]
            comm = rt.Comm(rank, N, local, 4 * rt.padded_elems(counts))
            base, _, scale = strat.partition("@")  # "mgwfbp@10": plan with 10x the calibrated a
            if base == "mgwfbp":
                sizes = [4096 << k for k in range(0, 20, 2) if (4096 << k) <= 4 * rt.padded_elems(counts)]
                if args.mode == "ce":  # the cost of one copy-engine push
                    meas = comm.calibrate_ce(sizes, warmup=2, reps=5)
                elif args.mode == "launch":  # the cost of one fused launch with launch_ctas CTAs
                    comm.set_max_ctas(args.launch_ctas)
                    meas = comm.calibrate(sizes, warmup=1, reps=3)
                    comm.set_max_ctas(0)
                else:
                    meas = comm.calibrate_engine(sizes, warmup=1, reps=3, engine_ctas=args.engine_ctas)
                t = torch.tensor([m.time_sec for m in meas], dtype=torch.float64, device=dev)
                if N > 1:
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                model_ab = gs.fit_model([gs.CommMeasurement(m.size_bytes, v) for m, v in zip(meas, t.tolist())])
                if scale:
                    model_ab = gs.AllReduceModel(model_ab.a * float(scale), model_ab.b)
                plan = gs.optimal_plan(trace, model_ab)
                D.agree_plan(plan.tags)
                extra = {"a_us": model_ab.a * 1e6, "b_ps_per_byte": model_ab.b * 1e12}
            elif base == "tuned":  # in-situ calibration of the plan (ddp.autotune_plan)
                from paper_1912_09268_b200.ddp import autotune_plan

                def tstep():
                    s_ = autotune_plan.current
                    s_.begin()
                    fwd_bwd(model)
                    s_.end()

                plan, tune = autotune_plan(model, comm, args.lr, trace, tstep, params=params,
                                           engine_ctas=args.engine_ctas, tail_groups=args.tail_groups,
                                           mode=args.mode, launch_ctas=args.launch_ctas)
                extra = {"autotune": {str(k): v for k, v in tune.items()}}
            elif base == "merged":  # every layer in one group, in this mode
                plan, extra = gs.MergePlan.all_merged(len(params)), {}
            elif strat == "wfbp":
                plan, extra = gs.MergePlan.all_normal(len(params)), {}
            else:
                plan, extra = gs.MergePlan.all_merged(len(params)), {}
            mode = "engine" if (strat == "single" and args.mode == "ce") else args.mode
            sync = MGWFBP(model, comm, args.lr, plan=plan, engine_ctas=args.engine_ctas, params=params,
                          tail_groups=args.tail_groups, mode=mode, launch_ctas=args.launch_ctas)
            if args.debug:
                import time
                for k in range(4):
                    t0 = time.time()
                    sync.begin()
                    fwd_bwd(model)
                    sync.end()
                    torch.cuda.synchronize()
                    print(f"[rank {rank}] {strat} debug step {k} {time.time() - t0:.3f}s", flush=True)
                sync.check()

            def step():
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
                sync.begin()
                fwd_bwd(model)
                sync.end()
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                phase_ev[-1].insert(0, e0)
                phase_ev[-1].append(e1)

            phase_ev.clear()
            ms = time_loop(step, args.iters, args.warmup)
            ph = phase_ev[-args.iters:]
            fwd = statistics.median(p[0].elapsed_time(p[1]) for p in ph)
            bwd = statistics.median(p[1].elapsed_time(p[2]) for p in ph)
            post = statistics.median(p[2].elapsed_time(p[3]) for p in ph)
            sync.check()
            results[strat] = {"iter_ms": ms, "host_ms": time_loop.host_ms, "groups": len(plan.groups()),
                              "fwd_ms": fwd, "bwd_ms": bwd, "post_bwd_ms": post, **extra}
            sync.close()
            comm.close()
        results[strat]["samples_per_s"] = N * args.batch / (results[strat]["iter_ms"] / 1e3)
        del model
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"model": args.model, "batch_per_gpu": args.batch, "n_gpus": N,
                          "mode": args.mode, "engine_ctas": args.engine_ctas, "launch_ctas": args.launch_ctas,
                          "tail_groups": args.tail_groups, "results": results}), flush=True)
    dist.destroy_process_group() if dist.is_initialized() else None


if __name__ == "__main__":
    main()
