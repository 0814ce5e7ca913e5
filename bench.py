"""MG-WFBP iteration benchmark on B200 (driver contract: one JSON line).

One step = one synchronous data-parallel iteration of the hot path on the
named model's layer trace: the backward pass replayed from B200-measured
per-tensor times (traces/<model>.json) on a compute stream, and every merge
group's fused pack -> NVLink all-reduce -> unpack+SGD kernel launched on a
comm stream the moment its head layer is ready (paper Algorithm 2), the
whole iteration one CUDA graph. Gradients are synthetic uniform[-1,1) fp32
(seed 0x5EED0000 + rank), weights uniform (seed 0xC0FFEE), lr 0.01.

  value   = N * K / (max over ranks of the device time of K MG-WFBP
            iterations)  [worker-iterations/s; driver scaling efficiency =
            value_N / (N * value_1) = t_iter(1) / t_iter(N), the paper's]
  plan    = optimal_plan(trace, (a, b)) with (a, b) fitted (fit_model) to
            an on-box calibration sweep of the same fused kernel at this N
  strategies: MG-WFBP (optimal), WFBP (all normal), single buffer (all
            merged), greedy (paper Algorithm 1) on the same pipeline

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--trace googlenet]
       python bench.py --impl reference ...   (CPU Algorithm 2 on host cores)
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (one rank per GPU).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "iter time & scaling eff. @1/2/4/8 B200 vs WFBP; merged allreduce bus GB/s"
UNIT = "worker-iters/s"
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction, /opt/skills/guides/B200_PROFILING.md
HBM_FALLBACK_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mgwfbp", choices=["mgwfbp", "reference"])
    ap.add_argument("--trace", default="googlenet")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--algo", default="auto", choices=["auto", "oneshot", "twoshot"])
    ap.add_argument("--oneshot-max", type=int, default=0, help="0: the library default for N")
    ap.add_argument("--cost", default="linear", choices=["linear", "table"],
                    help="linear: the reference's a + b*M (bit-exact optimal_plan); table: B200 extension, the same "
                         "DP on the calibration's piecewise measured curve")
    ap.add_argument("--tb-scale", type=float, default=1.0,
                    help="scale the trace's forward/backward times (emulates faster compute / smaller batches: "
                         "the comm-bound regime of the paper); 1.0 = the B200-measured trace")
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"],
                    help="gradient / merge-arena type (bf16: fp32 accumulation, fp32 master weights)")
    ap.add_argument("--engine-ctas", type=int, default=-1,
                    help="-1: persistent comm engine, one CTA per SM; >0: that many CTAs; "
                         "0: one fused kernel launch per group")
    ap.add_argument("--l2-flush-mib", type=int, default=256)
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--model", default="",
                    help="A_US,B_PS_PER_BYTE: skip the calibration and plan with this (a, b) "
                         "(ncu runs, where a calibration under kernel serialisation is meaningless)")
    return ap.parse_args()


def trace_path(name: str) -> str:
    return name if name.endswith(".json") else os.path.join(ROOT, "traces", f"{name}.json")


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        finally:
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# -------------------------------------------------------------- CPU legs
def cpu_pipeline_sample(trace, tags, P, lr, threads, budget_s, iters_cap=None):
    """The CPU restatement of Algorithm 2 (oracle port) on host buffers."""
    import numpy as np

    from oracle import pyoracle

    counts = [l.params for l in trace.layers]
    rng = np.random.default_rng(0x5EED0000)
    g = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    w = [[np.full(c, 0.5, np.float32) for c in counts] for _ in range(P)]
    t_b = [l.backward_time for l in trace.layers]
    first = pyoracle.pipeline_run(g, w, counts, t_b, trace.forward_time, tags, lr, threads, 1)[0]
    iters = max(3, min(200, int(budget_s / max(first, 1e-6))))
    if iters_cap is not None:
        iters = min(iters, iters_cap)
    times = pyoracle.pipeline_run(g, w, counts, t_b, trace.forward_time, tags, lr, threads, iters)
    return times


def ref_solver_us(trace, model, reps=200):
    import ctypes

    from oracle import pyoracle

    if pyoracle.REF is None:
        return None
    params = [l.params for l in trace.layers]
    t_b = [l.backward_time for l in trace.layers]
    L = len(params)
    p = (ctypes.c_uint64 * L)(*params)
    tb = (ctypes.c_double * L)(*t_b)
    out = (ctypes.c_uint8 * L)()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        pyoracle.REF.ref_optimal_plan(p, tb, L, trace.forward_time, trace.bytes_per_element, model.a, model.b, out)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


def cpu_path_detail(trace, model, budget_s=3.0):
    """SURVEY §8d "CPU path timed beside it": the reference's own solver and
    predictor on 1 core (oracle/_ref, the unmodified headers) and the CPU
    restatement of the merged all-reduce + SGD for config 1 (ResNet-50-sized,
    2 ranks as host buffers) on 1 core."""
    import ctypes
    import platform

    import numpy as np

    from oracle import pyoracle

    out = {"host": platform.processor() or platform.machine(), "nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            out["host"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    params = [l.params for l in trace.layers]
    t_b = [l.backward_time for l in trace.layers]
    L = len(params)
    p = (ctypes.c_uint64 * L)(*params)
    tb = (ctypes.c_double * L)(*t_b)
    tags = (ctypes.c_uint8 * L)()
    if pyoracle.REF is not None:
        def med(fn, reps=100):
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            return statistics.median(ts) * 1e6
        args = (p, tb, L, trace.forward_time, trace.bytes_per_element, model.a, model.b)
        out["ref_optimal_plan_us_1core"] = med(lambda: pyoracle.REF.ref_optimal_plan(*args, tags))
        out["ref_greedy_plan_us_1core"] = med(lambda: pyoracle.REF.ref_greedy_plan(*args, tags))
        it, nonov = ctypes.c_double(), ctypes.c_double()
        out["ref_iteration_time_us_1core"] = med(
            lambda: pyoracle.REF.ref_iteration_time(*args, tags, ctypes.byref(it), ctypes.byref(nonov)))
    # config 1: ResNet-50-sized merged all-reduce + SGD, 2 ranks, 1 core
    rng = np.random.default_rng(1)
    counts = [25_557_032]
    g = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(2)]
    w = [[np.full(c, 0.5, np.float32) for c in counts] for _ in range(2)]
    ts = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or not ts:
        t0 = time.perf_counter()
        pyoracle.allreduce_sgd(g, w, [0], 0.01)
        ts.append(time.perf_counter() - t0)
    out["allreduce_sgd_r50_2ranks_ms_1core"] = statistics.median(ts) * 1e3
    out["allreduce_sgd_r50_2ranks_GBps_1core"] = 2 * 4 * counts[0] * 3 / statistics.median(ts) / 1e9
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port of Algorithm 2
    + the reference's own optimal_plan from oracle/_ref) on host cores."""
    from paper_1912_09268_b200 import dist as D
    from paper_1912_09268_b200 import gradsched as gs

    rank, world, _ = D.env_world()
    if rank != 0:
        return 0
    N = max(world, args.gpus)
    trace = gs.load_trace(trace_path(args.trace))
    if args.tb_scale != 1.0:
        trace.forward_time *= args.tb_scale
        for l in trace.layers:
            l.backward_time *= args.tb_scale
    # paper cluster-independent model: a NVLink-class guess; the plan only
    # decides grouping, the CPU work is the same bytes either way
    model = gs.AllReduceModel(20e-6, 1.0 / 600e9)
    plan = gs.optimal_plan(trace, model)
    tags = [int(t) for t in plan.tags]
    threads = os.cpu_count() or 1
    cpu_pipeline_sample(trace, tags, N, args.lr, threads, 0.0, iters_cap=args.warmup)
    times = cpu_pipeline_sample(trace, tags, N, args.lr, threads, 1e9, iters_cap=args.steps)
    total = sum(times)
    value = N * len(times) / total
    solver = ref_solver_us(trace, model)
    sample = (f"{len(times)} CPU iterations of {args.trace} ({trace.n_layers()} tensors, "
              f"{trace.total_params()} fp32 params), {N} ranks emulated as host buffers; "
              f"reference optimal_plan {solver:.1f} us on 1 core" if solver else "")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": len(times),
        "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "impl": "reference",
        "data": "synthetic uniform[-1,1) fp32 gradients",
        "config": {"workload": args.trace, "trace": os.path.relpath(trace_path(args.trace), ROOT),
                   "plan": "optimal", "ranks": N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- GPU leg
def fit_with_fallback(gs, meas):
    try:
        return gs.fit_model(meas), "fit_model over the full sweep"
    except gs.FitError:
        small = [m for m in meas if m.size_bytes <= 4 << 20]
        try:
            return gs.fit_model(small), "fit_model over sizes <= 4 MiB (full sweep not linear)"
        except gs.FitError:
            t0 = min(m.time_sec for m in meas)
            big = sorted(meas, key=lambda m: m.size_bytes)[-2:]
            b = max(0.0, (big[1].time_sec - big[0].time_sec) / max(1, big[1].size_bytes - big[0].size_bytes))
            return gs.AllReduceModel(t0, b), "min-time startup + large-message slope"


def calibration_sizes(total_bytes: int, arena_bytes: int):
    top = min(arena_bytes, max(1 << 22, 1 << math.ceil(math.log2(max(total_bytes, 1)))))
    sizes = []
    s = 4096
    while s <= top:
        sizes.append(s)
        mid = int(s * math.sqrt(2)) & ~15
        if mid < top:
            sizes.append(mid)
        s *= 2
    return sizes


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    from paper_1912_09268_b200 import dist as D
    from paper_1912_09268_b200 import gradsched as gs
    from paper_1912_09268_b200 import runtime as rt

    rank, world, local = D.init("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N = world
    trace = gs.load_trace(trace_path(args.trace))
    if args.tb_scale != 1.0:
        trace.forward_time *= args.tb_scale
        for l in trace.layers:
            l.backward_time *= args.tb_scale
    bf16 = args.dtype == "bf16"
    esz = 2 if bf16 else 4
    gdt = torch.bfloat16 if bf16 else torch.float32
    trace.bytes_per_element = esz  # the planner costs groups in gradient bytes (trace.hpp:50)
    counts = [l.params for l in trace.layers]
    L = len(counts)
    total_bytes = esz * sum(counts)
    padded = rt.padded_elems(counts, rt.BF16 if bf16 else rt.F32)
    granule = 16 // esz

    # gradients: one flat buffer (16-byte aligned layer views, like a
    # framework's flat grad buffer); weights: fp32, one allocation per layer
    gen = torch.Generator(device=dev)
    gen.manual_seed(0x5EED0000 + rank)
    flat_grad = torch.empty(padded, dtype=torch.float32, device=dev).uniform_(-1, 1, generator=gen).to(gdt)
    offs = [0]
    for c in counts:
        offs.append(offs[-1] + (c + granule - 1) // granule * granule)
    grads = [flat_grad[offs[i]:offs[i] + counts[i]] for i in range(L)]
    wgen = torch.Generator(device=dev)
    wgen.manual_seed(0xC0FFEE)
    weights = [torch.empty(max(c, 1), dtype=torch.float32, device=dev).uniform_(-1, 1, generator=wgen)[:c]
               for c in counts]

    comm = rt.Comm(rank, N, local, 4 * max(padded, 1 << 20))
    if args.oneshot_max > 0:
        comm.set_oneshot_max(args.oneshot_max)

    # ---- N1: on-box calibration of the fused kernel at this N, fitted
    sizes = calibration_sizes(total_bytes, 4 * padded)
    if args.model:
        a_us, b_ps = (float(x) for x in args.model.split(","))
        sizes = sizes[:2]  # (a short sweep still exercises the calibration kernels)
    if args.engine_ctas != 0:
        meas = comm.calibrate_engine(sizes, warmup=3, reps=15, algo=args.algo, engine_ctas=args.engine_ctas,
                                     dtype=rt.BF16 if bf16 else rt.F32)
    else:
        meas = comm.calibrate(sizes, warmup=3, reps=15, algo=args.algo)
    tvec = torch.tensor([m.time_sec for m in meas], dtype=torch.float64, device=dev)
    if N > 1:
        torch.distributed.all_reduce(tvec, op=torch.distributed.ReduceOp.MAX)
    meas = [gs.CommMeasurement(m.size_bytes, float(t)) for m, t in zip(meas, tvec.tolist())]
    model, fit_how = fit_with_fallback(gs, meas)
    if args.model:
        model, fit_how = gs.AllReduceModel(a_us * 1e-6, b_ps * 1e-12), "given by --model (not calibrated)"
    out_dir = os.environ.get("MGW_OUT_DIR")
    if out_dir and rank == 0:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, f"calib_{args.trace}_P{N}.csv"), "w") as f:
            f.write("size_bytes,time_us\n")
            for m in meas:
                f.write(f"{m.size_bytes},{m.time_sec * 1e6:.3f}\n")

    # ---- plans (host solver, replicated; verified identical across ranks)
    plans = {
        "mgwfbp": gs.optimal_plan(trace, model) if args.cost == "linear" else gs.optimal_plan_table(trace, meas),
        "wfbp": gs.MergePlan.all_normal(L),
        "single_buffer": gs.MergePlan.all_merged(L),
        "greedy": gs.greedy_plan(trace, model),
    }
    digest = D.agree_plan(plans["mgwfbp"].tags)
    flush = args.l2_flush_mib << 20
    pipes = {}
    dplans = {}
    for name, plan in plans.items():
        dplans[name] = rt.DevicePlan(comm, grads, weights, plan)
        pipes[name] = rt.Pipeline(dplans[name], trace, args.lr, args.algo,
                                  record_group_times=True, l2_flush_bytes=flush,
                                  engine_ctas=args.engine_ctas)
    # the headline pipeline: the same plan without the per-group timing
    # stamps (an instrumented twin above supplies group times / the tail)
    pipes["headline"] = rt.Pipeline(dplans["mgwfbp"], trace, args.lr, args.algo, record_group_times=False,
                                    l2_flush_bytes=flush, engine_ctas=args.engine_ctas)

    def timed(name, iters):
        D.barrier()
        torch.cuda.synchronize()
        ms = pipes[name].run(iters)
        torch.cuda.synchronize()
        D.barrier()
        return ms

    for name in pipes:
        pipes[name].run(max(1, args.warmup))
    torch.cuda.synchronize()

    # ---- the timed region: K MG-WFBP iterations
    launches0 = rt.kernel_launches()
    with ClockSampler(local) as clk:
        ms = timed("headline", args.steps)
    launches = rt.kernel_launches() - launches0
    clocks = clk.summary()
    t_total = D.max_over_ranks(sum(ms) / 1e3, dev)
    value = N * args.steps / t_total

    # ---- comparison strategies on the same box / pipeline
    strat = {}
    for name in ("mgwfbp", "wfbp", "single_buffer", "greedy"):
        m = timed(name, args.steps)  # instrumented pipelines, alike for every strategy
        per = sorted(m)
        med = D.max_over_ranks(statistics.median(per), dev)
        p10 = D.max_over_ranks(per[max(0, int(0.1 * len(per)) - 0)], dev)
        p90 = D.max_over_ranks(per[min(len(per) - 1, int(0.9 * len(per)))], dev)
        pred = (gs.iteration_time(trace, plans[name], model).iteration_time if args.cost == "linear"
                else gs.iteration_time_table(trace, plans[name], meas))
        strat[name] = {"iter_ms_median": med, "iter_ms_p10": p10, "iter_ms_p90": p90,
                       "predicted_ms": pred * 1e3, "groups": dplans[name].n_groups}
        if args.engine_ctas != 0:
            # device clock of the last iteration: exposed comm after the replay
            tl = pipes[name].device_timeline()
            strat[name]["device_tail_us"] = D.max_over_ranks(tl["tail_us"], dev)
            strat[name]["device_replay_ms"] = tl["replay_us"] / 1e3
        if name == "mgwfbp":
            group_ms = pipes["mgwfbp"].group_times_ms()
    compute_ms = (trace.forward_time + sum(l.backward_time for l in trace.layers)) * 1e3

    # ---- e2e through the public API with host buffers
    # Each step: the step's gradients H2D from pinned host memory (captured in
    # the iteration graph on the comm branch, overlapping the forward replay;
    # every group kernel waits for it) and 16 result bytes D2H at the end.
    host_grad = torch.empty(padded, dtype=gdt, pin_memory=True)
    host_grad.copy_(flat_grad.cpu())
    host_out = torch.empty(4, dtype=torch.float32, pin_memory=True)
    out_src = weights[0][:4] if counts[0] >= 4 else flat_grad[:4]
    pipe = rt.Pipeline(dplans["mgwfbp"], trace, args.lr, args.algo, record_group_times=False,
                       l2_flush_bytes=flush, engine_ctas=args.engine_ctas,
                       h2d=(host_grad, flat_grad), d2h=(host_out, out_src))
    pipe.run(max(1, args.warmup))
    D.barrier()
    torch.cuda.synchronize()
    e2e_ms = pipe.run(args.steps)
    e2e_s = D.max_over_ranks(sum(e2e_ms) / 1e3, dev)
    D.barrier()
    pipes["e2e"] = pipe

    # ---- roofline of the dominant kernel (the fused group kernel)
    peaks = measured_peaks()
    gbytes = [dplans["mgwfbp"].group_span(g)[2] for g in range(dplans["mgwfbp"].n_groups)]
    kern_s = sum(group_ms) / 1e3
    w_per_g = 4 / esz  # fp32 weight bytes per gradient byte
    if N == 1:
        algo_bytes = sum((1 + 2 * w_per_g) * b for b in gbytes)  # read grad, read W, write W
        peak = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
        roof = {"bound": "hbm", "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
    else:
        algo_bytes = sum(2 * (N - 1) / N * b for b in gbytes)  # NVLink bus bytes
        peak = NVLINK_PEER_GBS
        roof = {"bound": "nvlink", "peak_source": "measured B200 peer copy 770 GB/s/direction (B200_PROFILING.md)"}
    achieved = algo_bytes / kern_s / 1e9 if kern_s > 0 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.trace}_P{N}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    # the same fused kernel on the LARGEST calibrated group (cold L2, one
    # group on an idle engine): bytes that cross the bound / its time — the
    # bandwidth regime, next to the latency-dominated per-iteration figure
    per_byte = (1 + 2 * w_per_g) if N == 1 else 2 * (N - 1) / N
    big_m = max(meas, key=lambda m: m.size_bytes)
    asym = per_byte * big_m.size_bytes / big_m.time_sec / 1e9 if big_m.time_sec > 0 else None
    roof.update({"kernel": ("engine_kernel/run_group (fused pack + push all-reduce + unpack/SGD), "
                            "per-group %globaltimer stamps" if args.engine_ctas
                            else "group_allreduce_kernel (fused pack + push all-reduce + unpack/SGD)"),
                 "achieved": achieved, "peak": peak, "unit": "GB/s",
                 "frac": achieved / peak if achieved else None, "traffic": traffic,
                 "traffic_evidence": (
                     "profiles/r1_ncu_hbm_kernels_256MiB.txt: the P=1 fused group kernel (same run_group code as "
                     "the engine) moves 752 MB DRAM vs 805 MB algorithmic per 256 MiB launch (no re-reads)"
                     if N == 1 else
                     "profiles/r1_ncu_loopback_twoshot_64MiB.txt: the two-shot data path in loopback moves "
                     "623 MB DRAM vs 671 MB algorithmic (P=2, 64 MiB/rank; no re-reads)")
                     + "; the engine kernel itself cannot run under ncu's serialisation (it waits on the replay)",
                 "algorithmic_bytes_per_iter": algo_bytes, "kernel_ms_per_iter": kern_s * 1e3,
                 "launches_per_iter": len(group_ms),
                 "note": f"small groups are latency-bound ({args.trace}: {sum(counts)} params over "
                         f"{len(group_ms)} groups); the bandwidth regime is the largest_group row",
                 "largest_group": {"achieved": asym, "frac": asym / peak if asym else None,
                                   "group_bytes": big_m.size_bytes, "us": big_m.time_sec * 1e6,
                                   "from": "the largest size of the on-box calibration sweep"}})

    # merged all-reduce bus GB/s = 2(P-1)/P * S / t: ours (fused kernel, from
    # the calibration sweep) next to NCCL (torch.distributed.all_reduce, same
    # sizes, comparison baseline only)
    bus = {}
    if N > 1:
        big = [m for m in meas if m.size_bytes >= (1 << 20)]
        ncclt = []
        for m in big:
            x = torch.ones(m.size_bytes // esz, dtype=gdt, device=dev)
            for _ in range(3):
                torch.distributed.all_reduce(x)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            ev[0].record()
            for _ in range(10):
                torch.distributed.all_reduce(x)
            ev[1].record()
            ev[1].synchronize()
            ncclt.append(D.max_over_ranks(ev[0].elapsed_time(ev[1]) / 10 / 1e3, dev))
            del x
        for m, tn in zip(big, ncclt):
            f = 2 * (N - 1) / N * m.size_bytes / 1e9
            bus[str(m.size_bytes)] = {"mgwfbp": f / m.time_sec, "nccl": f / tn}

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        times = cpu_pipeline_sample(trace, [int(t) for t in plans["mgwfbp"].tags], 1, args.lr, threads,
                                    args.cpu_budget_s)
        solver = ref_solver_us(trace, model)
        detail = cpu_path_detail(trace, model)
        cpu = {"value": len(times) / sum(times), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{len(times)} iterations of the CPU Algorithm-2 restatement (oracle/mgw_oracle.c, "
                         f"same trace/plan, P=1, {threads} threads)"
                         + (f"; reference optimal_plan (oracle/_ref) {solver:.1f} us on 1 core" if solver else "")
                         + ("; the CPU path reduces fp32 gradients (no bf16 CPU pipeline)" if bf16 else ""),
               "detail": detail}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_total / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": (f"synthetic uniform[-1,1) {args.dtype} gradients"
                     + (" (fp32 accumulation, fp32 master weights)" if bf16 else "")
                     + "; backward replayed from B200-measured per-tensor t_b"),
            "config": {"workload": args.trace, "trace": os.path.relpath(trace_path(args.trace), ROOT),
                       "layers": L, "params": sum(counts), "grad_bytes": total_bytes,
                       "plan": ("optimal_plan on on-box calibrated (a, b)" if args.cost == "linear" else
                                "optimal_plan_table on the on-box calibration curve (B200 extension)"),
                       "plan_sha256": digest[:16],
                       "groups": dplans["mgwfbp"].n_groups, "algo": args.algo, "oneshot_max": comm.oneshot_max,
                       "comm": ("persistent engine, %s CTAs" % ("1/SM" if args.engine_ctas < 0 else args.engine_ctas))
                               if args.engine_ctas else "one fused kernel launch per group",
                       "parallelism": f"dp{N}", "l2": f"flushed every iteration ({args.l2_flush_mib} MiB memset "
                                                     "on the comm stream during the forward replay)",
                       "compute_ms": compute_ms, "tb_scale": args.tb_scale},
            "calibration": {"a_us": model.a * 1e6, "b_ps_per_byte": model.b * 1e12, "how": fit_how,
                            "sizes": len(meas), "largest_bytes": meas[-1].size_bytes,
                            "largest_us": meas[-1].time_sec * 1e6},
            "strategies": strat,
            "speedup_vs_wfbp": strat["wfbp"]["iter_ms_median"] / strat["mgwfbp"]["iter_ms_median"],
            "speedup_vs_single_buffer": strat["single_buffer"]["iter_ms_median"] / strat["mgwfbp"]["iter_ms_median"],
            "bus_gbs": bus,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": N * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": padded * esz,
                    "d2h_bytes_per_step": 16},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    # Teardown order matters: pinned host blocks used on the pipeline's
    # stream must be released while that stream still exists.
    torch.cuda.synchronize()
    del host_grad, host_out
    import gc

    gc.collect()
    torch._C._host_emptyCache()
    for p in pipes.values():
        p.close()
    for p in dplans.values():
        p.close()
    comm.close()
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
