"""MG-WFBP iteration benchmark on B200 (driver contract: one JSON line).

One step = one synchronous data-parallel iteration of the hot path on the
named model's layer trace (default BERT-large, BASELINE config 5, the largest
config that fits one B200): the backward pass replayed from B200-measured
per-tensor times (traces/<model>.json) on a compute stream, and every merge
group's fused pack -> NVLink all-reduce -> unpack+SGD run by the persistent
comm engine the moment its head layer is ready (paper Algorithm 2), the
whole iteration one CUDA graph. Gradients are synthetic uniform[-1,1) fp32
(seed 0x5EED0000 + rank), weights uniform (seed 0xC0FFEE), lr 0.01.

  value   = N * K / (max over ranks of the device time of K MG-WFBP
            iterations)  [worker-iterations/s; driver scaling efficiency =
            value_N / (N * value_1) = t_iter(1) / t_iter(N), the paper's]
  plan    = optimal_plan(trace, fit_model(committed on-box calibration
            profiles/calib/calib_<trace>_P<N>.csv)) — the SAME plan in both
            arms (same plan_sha256, identical config); the live on-box sweep
            of this run is reported beside it (calibration.onbox)
  strategies: MG-WFBP (optimal), WFBP (all normal), single buffer (all
            merged), greedy (paper Algorithm 1) on the same pipeline
  roofline: the engine kernel in standalone drain (every group ready), CUDA
            events per launch: algorithmic bytes / launch time vs HBM (N=1)
            or NVLink 900 GB/s per direction (N>1)

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--trace bert_large]
       python bench.py --impl reference ...   (the reference's CPU path: its
           own optimal_plan from oracle/_ref + the CPU Algorithm-2 port; never
           imports this package)
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (one rank per GPU).
"""
from __future__ import annotations

import argparse
import glob
import hashlib
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
# The other-protocol diagnostics (drain + bus columns) run where both
# protocols were validated over real NVLink (N = 2, 4); at N = 8 the bench
# runs the default path only (P = 8 is validated in loopback).
OTHER_PROTOCOL_MAX_N = 4
NVLINK_GBS = 900.0       # NVLink 5 per direction (north_star / BASELINE.md §3 denominator)
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction, /opt/skills/guides/B200_PROFILING.md (secondary)
HBM_FALLBACK_GBS = 6650.0
L2_BYTES = 126 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # >= 200 timed iterations after 20 warm-up
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="mgwfbp", choices=["mgwfbp", "reference"])
    ap.add_argument("--trace", default="bert_large")
    ap.add_argument("--plan-source", default="committed", choices=["committed", "onbox"],
                    help="committed: both arms plan from profiles/calib/calib_<trace>_P<N>.csv (same plan); "
                         "onbox: the GPU arm plans from this run's own calibration sweep")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--algo", default="auto", choices=["auto", "oneshot", "twoshot"])
    ap.add_argument("--oneshot-max", type=int, default=0, help="0: the library default for N")
    ap.add_argument("--nvls", type=float, default=0.0,
                    help="MiB: route fp32 standalone group launches of at least this size through the NVLS "
                         "(switch-reduced) variant (N > 1 only; 0: off, the default). A negative value sets "
                         "NVLS up for the bus_gbs table only (measured beside NCCL), data path unchanged.")
    ap.add_argument("--cost", default="linear", choices=["linear", "table"],
                    help="linear: the reference's a + b*M (bit-exact optimal_plan); table: B200 extension, the same "
                         "DP on the calibration's piecewise measured curve")
    ap.add_argument("--tb-scale", type=float, default=1.0,
                    help="scale the trace's forward/backward times (emulates faster compute / smaller batches: "
                         "the comm-bound regime of the paper); 1.0 = the B200-measured trace")
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"],
                    help="gradient / merge-arena type (bf16: fp32 accumulation, fp32 master weights)")
    ap.add_argument("--protocol", default="auto", choices=["auto", "chunked", "stream"],
                    help="fused all-reduce protocol at N > 1: auto (the library default: chunked), chunked "
                         "(per-chunk cross-rank barriers) or stream (per-tile delivery counts in the engine, the "
                         "last-ready group as a chunked launch)")
    ap.add_argument("--stream-batches", default="",
                    help="CREDIT,AG: streamed-protocol publication batches (default: the library's 8,4)")
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


# ------------------------------------------- shared by both arms (no package)
def load_trace_json(path: str, tb_scale: float = 1.0) -> dict:
    """The reference's load_trace (trace.hpp:148-219) restated for the
    reference arm, which must not load this package: microseconds / 1e6 on
    correctly rounded parses (Python's float() and nlohmann's strtod agree),
    so the doubles equal the library's ModelTrace bit for bit."""
    with open(path) as f:
        d = json.load(f)
    tr = {"names": [l["name"] for l in d["layers"]],
          "params": [int(l["params"]) for l in d["layers"]],
          "t_b": [float(l["backward_time_us"]) / 1e6 for l in d["layers"]],
          "t_f": float(d["forward_time_us"]) / 1e6,
          "bpe": int(d.get("bytes_per_element", 4))}
    if tb_scale != 1.0:
        tr["t_f"] *= tb_scale
        tr["t_b"] = [t * tb_scale for t in tr["t_b"]]
    return tr


def committed_calibration(trace_name: str, N: int):
    """profiles/calib/calib_<trace>_P<N>.csv — an on-box calibration sweep
    of the fused engine kernel committed from an earlier run on this box type
    (P8: projected from P4, profiles/calib/README.md). Both arms fit it with
    the reference's fit_model, so they plan identically."""
    rel = os.path.join("profiles", "calib", f"calib_{os.path.basename(trace_name).replace('.json', '')}_P{N}.csv")
    return rel if os.path.exists(os.path.join(ROOT, rel)) else None


def plan_digest(tags) -> str:
    return hashlib.sha256(bytes(int(t) for t in tags)).hexdigest()


def common_config(name: str, tr: dict, N: int, tags, calib_rel, tb_scale: float, dtype: str) -> dict:
    """The `config` object, built identically by both arms from the trace
    file, the plan's tags and the calibration path."""
    esz = 2 if dtype == "bf16" else 4
    total = sum(tr["params"])
    inputs = 2 * esz * total
    return {
        "workload": name, "trace": os.path.relpath(trace_path(name), ROOT), "layers": len(tr["params"]),
        "params": total, "grad_bytes": esz * total, "dtype": dtype,
        "plan": "optimal_plan (reference planner.hpp:63-98) on fit_model of " + (calib_rel or "?"),
        "calibration_csv": calib_rel, "plan_sha256": plan_digest(tags)[:16],
        "groups": sum(1 for i, t in enumerate(tags) if i == 0 or int(t) == 0),
        "parallelism": f"dp{N}", "ranks": N,
        "compute_ms": (tr["t_f"] + sum(tr["t_b"])) * 1e3, "tb_scale": tb_scale,
        "l2": ("inputs (gradients + weights, %.0f MB per rank) exceed the 126 MB L2; " % (inputs / 1e6)
               if inputs > L2_BYTES else "inputs fit in L2; ") + "the GPU arm also evicts L2 every iteration",
    }


def host_info() -> dict:
    import platform

    out = {"host": platform.processor() or platform.machine(), "nproc": os.cpu_count(),
           "isa": platform.machine()}
    try:
        with open("/proc/cpuinfo") as f:
            out["host"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    return out


# -------------------------------------------------------------- CPU legs
def ref_lib():
    """oracle/_ref: the reference headers compiled unmodified (None when the
    reference was not available to build it) and the C restatement."""
    from oracle import pyoracle

    return pyoracle


def ref_fit(csv_path: str):
    """(a, b) by the reference's own load_measurements_csv + fit_model
    (comm_model.hpp:209-308) from oracle/_ref; the C restatement otherwise."""
    import ctypes

    po = ref_lib()
    if po.REF is not None:
        a, b = ctypes.c_double(), ctypes.c_double()
        rc = po.REF.ref_fit_csv(csv_path.encode(), ctypes.byref(a), ctypes.byref(b))
        if rc != 0:
            raise RuntimeError(f"reference fit_model failed on {csv_path}")
        return a.value, b.value, "reference"
    rows = []
    with open(csv_path) as f:
        next(f)
        for line in f:
            sz, us = line.strip().split(",")
            rows.append((int(sz), float(us) / 1e6))
    a, b = po.orc_fit([r[0] for r in rows], [r[1] for r in rows])
    return a, b, "port"


def ref_plan(tr: dict, a: float, b: float, bpe: int):
    po = ref_lib()
    if po.REF is not None:
        return po.ref_optimal(tr["params"], tr["t_b"], tr["t_f"], bpe, a, b), "reference"
    return po.orc_optimal(tr["params"], tr["t_b"], tr["t_f"], bpe, a, b), "port"


def cpu_pipeline_sample(tr: dict, tags, P, lr, threads, budget_s, iters_cap=None):
    """The CPU restatement of Algorithm 2 (oracle port) on host buffers."""
    import numpy as np

    po = ref_lib()
    counts = tr["params"]
    rng = np.random.default_rng(0x5EED0000)
    g = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    w = [[np.full(c, 0.5, np.float32) for c in counts] for _ in range(P)]
    first = po.pipeline_run(g, w, counts, tr["t_b"], tr["t_f"], tags, lr, threads, 1)[0]
    iters = max(3, min(200, int(budget_s / max(first, 1e-6))))
    if iters_cap is not None:
        iters = min(iters, iters_cap)
    return po.pipeline_run(g, w, counts, tr["t_b"], tr["t_f"], tags, lr, threads, iters)


def _median_us(fn, reps=1000, cap_s=1.0):
    ts = []
    t_end = time.perf_counter() + cap_s
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end and len(ts) >= 50:
            break
    return statistics.median(ts) * 1e6, len(ts)


def solver_table(bpe: int = 4) -> dict:
    """BASELINE.md §3.1-3.2 on 1 host core: the reference's optimal_plan,
    greedy_plan and iteration_time (oracle/_ref, unmodified headers) on every
    trace at the committed on-box (a, b) of P = 2 / 4 / 8 — median of up to
    1000 runs (1 s cap per entry)."""
    import ctypes

    po = ref_lib()
    if po.REF is None:
        return {"unavailable": "oracle/_ref not built (the reference sources were not present at build time)"}
    out = {}
    names = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(ROOT, "traces", "*.json"))
                   if not p.endswith("META.json"))
    for name in names + ["skewed_161"]:
        path = (os.path.join(ROOT, "tests", "golden", "skewed_161.json") if name == "skewed_161"
                else trace_path(name))
        tr = load_trace_json(path)
        L = len(tr["params"])
        p = (ctypes.c_uint64 * L)(*tr["params"])
        tb = (ctypes.c_double * L)(*tr["t_b"])
        tags = (ctypes.c_uint8 * L)()
        row = {"layers": L}
        for P in (2, 4, 8):
            rel = committed_calibration("resnet50" if name == "skewed_161" else name, P)
            if rel is None:
                continue
            a, b, _ = ref_fit(os.path.join(ROOT, rel))
            args = (p, tb, L, tr["t_f"], bpe, a, b)
            opt, n1 = _median_us(lambda: po.REF.ref_optimal_plan(*args, tags))
            gre, _ = _median_us(lambda: po.REF.ref_greedy_plan(*args, tags))
            it, no = ctypes.c_double(), ctypes.c_double()
            pre, _ = _median_us(lambda: po.REF.ref_iteration_time(*args, tags, ctypes.byref(it), ctypes.byref(no)))
            row[f"P{P}"] = {"a_us": a * 1e6, "b_ps": b * 1e12, "optimal_plan_us": opt, "greedy_plan_us": gre,
                            "iteration_time_us": pre, "runs": n1}
        out[name] = row
    return out


def allreduce_cpu_config1(budget_s=3.0) -> dict:
    """Config 1's CPU merged all-reduce (ResNet-50-sized 25.6 M fp32, 2 ranks
    as host buffers: x 1/P, rank-order sum, SGD) on 1 core and on all cores
    (the C restatement's threaded pipeline, no replay wait)."""
    import numpy as np

    po = ref_lib()
    n = 25_557_032
    rng = np.random.default_rng(1)
    g = [[rng.uniform(-1, 1, n).astype(np.float32)] for _ in range(2)]
    w = [[np.full(n, 0.5, np.float32)] for _ in range(2)]
    ts = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or not ts:
        t0 = time.perf_counter()
        po.allreduce_sgd(g, w, [0], 0.01)
        ts.append(time.perf_counter() - t0)
    one = statistics.median(ts)
    threads = os.cpu_count() or 1
    allc = statistics.median(po.pipeline_run(g, w, [n], [0.0], 0.0, [0], 0.01, threads, 5))
    algo = 2 * 4 * n * 3  # per rank: read grad, read W, write W
    return {"ms_1core": one * 1e3, "GBps_1core": algo / one / 1e9, "ms_all_cores": allc * 1e3,
            "GBps_all_cores": algo / allc / 1e9, "threads": threads}


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores — its own
    fit_model + optimal_plan (oracle/_ref, the unmodified headers) on the
    committed calibration, and the CPU restatement of Algorithm 2 (oracle
    port: the reference has no runtime) with N ranks as host buffers. Never
    imports paper_1912_09268_b200 (its libmgwfbp.so stays unloaded)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    N = max(world, args.gpus)
    tr = load_trace_json(trace_path(args.trace), args.tb_scale)
    bpe = 2 if args.dtype == "bf16" else 4
    calib = committed_calibration(args.trace, N)
    if calib is None:
        print(json.dumps({"impl": "reference", "unavailable": f"no committed calibration for {args.trace} P{N}"}))
        return 0
    a, b, fit_kind = ref_fit(os.path.join(ROOT, calib))
    tags, plan_kind = ref_plan(tr, a, b, bpe)
    threads = os.cpu_count() or 1
    # bounded sample: at most --steps iterations and about a minute of CPU work
    # (N = 8 BERT-large reduces 8 x 1.34 GB per iteration on the host)
    cpu_pipeline_sample(tr, tags, N, args.lr, threads, 0.0, iters_cap=max(1, min(args.warmup, 3)))
    times = cpu_pipeline_sample(tr, tags, N, args.lr, threads, 60.0, iters_cap=args.steps)
    total = sum(times)
    value = N * len(times) / total
    ms = total / len(times) * 1e3
    cfg = common_config(args.trace, tr, N, tags, calib, args.tb_scale, args.dtype)
    sample = (f"{len(times)} CPU iterations of {args.trace} ({len(tags)} tensors, {sum(tr['params'])} fp32 params "
              f"per rank), {N} ranks emulated as host buffers, {threads} threads; plan by the {plan_kind} "
              f"optimal_plan on the {fit_kind} fit of {calib}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": len(times),
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "impl": "reference",
        "data": "synthetic uniform[-1,1) fp32 gradients",
        "config": cfg,
        "exposed_comm_ms": ms - cfg["compute_ms"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "host": host_info()},
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
    tr_json = load_trace_json(trace_path(args.trace), args.tb_scale)
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
    # every rank must have mapped every peer's arena over NVLink (P = 8:
    # 7 IPC peers) before anything runs
    peers = comm.num_peers()
    if peers != N:
        raise RuntimeError(f"rank {rank}: {peers} of {N} ranks mapped (CUDA IPC over NVLink)")
    if N > 1:
        print(f"[bench] rank {rank}/{N}: {peers} ranks mapped over NVLink (CUDA IPC)", file=sys.stderr, flush=True)
    if args.oneshot_max > 0:
        comm.set_oneshot_max(args.oneshot_max)
    if N > 1:
        comm.set_protocol(args.protocol)  # (P = 1 always runs the TMA-fed single-rank engine)
        if args.stream_batches:
            comm.set_stream_batches(*(int(x) for x in args.stream_batches.split(",")))
    # NVLS (switch-reduced two-shot, opt-in): --nvls X routes
    # groups >= X MiB through it; --nvls -1 only measures it (bus_gbs)
    nvls = "off" if N > 1 else "n/a (N = 1)"
    if N > 1 and not bf16 and args.nvls != 0:
        nvls = "unsupported on this pool"
        ok = torch.tensor([1.0 if comm.nvls_supported() else 0.0], device=dev)
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        if ok.item() > 0:
            comm.enable_nvls(int(max(args.nvls, 0.0) * (1 << 20)))
            nvls = (f"on for groups >= {args.nvls} MiB" if args.nvls > 0 else "measured only (bus_gbs)")

    # ---- N1: on-box calibration of the fused engine kernel at this N
    sizes = calibration_sizes(total_bytes, 4 * padded)
    if args.model:
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
    onbox_model, onbox_how = fit_with_fallback(gs, meas)
    out_dir = os.environ.get("MGW_OUT_DIR")
    if out_dir and rank == 0:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, f"calib_{args.trace}_P{N}.csv"), "w") as f:
            f.write("size_bytes,time_us\n")
            for m in meas:
                f.write(f"{m.size_bytes},{m.time_sec * 1e6:.3f}\n")

    # ---- the plan's cost model: the committed calibration (identical in
    # the reference arm) unless --plan-source onbox / --model
    calib = committed_calibration(args.trace, N)
    if args.model:
        a_us, b_ps = (float(x) for x in args.model.split(","))
        model, model_how = gs.AllReduceModel(a_us * 1e-6, b_ps * 1e-12), "given by --model (not calibrated)"
    elif args.plan_source == "committed" and calib is not None:
        model = gs.fit_model(gs.load_measurements_csv(os.path.join(ROOT, calib)))
        model_how = f"fit_model of the committed calibration {calib}"
    else:
        model, model_how, calib = onbox_model, "this run's on-box sweep: " + onbox_how, None

    # ---- plans (host solver, replicated; verified identical across ranks)
    plans = {
        "mgwfbp": gs.optimal_plan(trace, model) if args.cost == "linear" else gs.optimal_plan_table(trace, meas),
        "wfbp": gs.MergePlan.all_normal(L),
        "single_buffer": gs.MergePlan.all_merged(L),
        "greedy": gs.greedy_plan(trace, model),
    }
    onbox_plan = gs.optimal_plan(trace, onbox_model)
    digest = D.agree_plan(plans["mgwfbp"].tags)
    cfg = common_config(args.trace, tr_json, N, [int(t) for t in plans["mgwfbp"].tags], calib, args.tb_scale,
                        args.dtype)
    assert cfg["plan_sha256"] == digest[:16]
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
    ms_step = t_total / args.steps * 1e3

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
    compute_ms = (trace.forward_time + sum(l.backward_time for l in trace.layers)) * 1e3
    # iteration lower bound: max(compute, t_f + t_b of
    # the first layer the backward finishes + every group at its bus roofline)
    gb_plan = [dplans["mgwfbp"].group_span(g)[2] for g in range(dplans["mgwfbp"].n_groups)]
    roof_comm_s = sum(2 * (N - 1) / N * b for b in gb_plan) / (NVLINK_GBS * 1e9)
    bound_ms = max(compute_ms, (trace.forward_time + trace.layers[-1].backward_time + roof_comm_s) * 1e3)

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

    # ---- roofline of the dominant kernel: the persistent engine draining
    # the whole plan (every group ready at launch), CUDA events per launch on
    # the engine's stream, L2 evicted before each launch
    peaks = measured_peaks()
    gbytes = [dplans["mgwfbp"].group_span(g)[2] for g in range(dplans["mgwfbp"].n_groups)]
    roof = {}
    engine_protocol = "none (one launch per group)"
    if args.engine_ctas != 0:
        D.barrier()
        engine_protocol = pipes["headline"].engine_protocol
        drain = pipes["headline"].drain(max(3, min(args.steps, 20)))
        kern_s = D.max_over_ranks(statistics.mean(drain) / 1e3, dev)
        w_per_g = 4 / esz  # fp32 weight bytes per gradient byte
        hbm_bytes = sum((1 + 2 * w_per_g) * b for b in gbytes)  # read grad, read W, write W
        if N == 1:
            algo_bytes = hbm_bytes
            peak = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
            roof = {"bound": "hbm", "peak_source": ("MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks
                                                    else "B200_PROFILING.md fallback"),
                    "peak_note": "the peak is a 1:1 read:write copy; the drain's traffic is 2 reads : 1 write "
                                 "(grad + W in, W out), which HBM serves up to ~1 % faster, so frac can "
                                 "exceed 1; frac_vs_nominal is against the 7.7 TB/s HGX B200 figure",
                    "frac_vs_nominal": None}
        else:
            algo_bytes = sum(2 * (N - 1) / N * b for b in gbytes)  # NVLink bus bytes per rank per direction
            peak = NVLINK_GBS
            roof = {"bound": "nvlink", "peak_source": "NVLink 5 900 GB/s per direction (north_star); "
                                                      "frac_vs_770 = the measured peer-copy figure"}
        achieved = algo_bytes / kern_s / 1e9
        if N == 1:
            roof["frac_vs_nominal"] = achieved / 7700.0
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"traffic_{args.trace}_P{N}.json")
        if os.path.exists(prof):
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        per_byte = (1 + 2 * w_per_g) if N == 1 else 2 * (N - 1) / N
        big_m = max(meas, key=lambda m: m.size_bytes)
        asym = per_byte * big_m.size_bytes / big_m.time_sec / 1e9 if big_m.time_sec > 0 else None
        roof.update({
            "kernel": f"engine_kernel<{N},{'bf16' if bf16 else 'float'}> standalone drain: the whole plan's fused "
                      f"pack -> all-reduce -> unpack+SGD, every group ready at launch",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "traffic_source": (os.path.relpath(prof, ROOT) + " (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                               "of the same drain launch)") if traffic else None,
            "algorithmic_bytes_per_launch": algo_bytes, "hbm_algorithmic_bytes_per_launch": hbm_bytes,
            "bytes_formula": ("3*S fp32 (read grad, read W, write W)" if N == 1 else
                              "2(P-1)/P*S NVLink bus bytes per rank per direction"),
            "launch_ms_mean": kern_s * 1e3, "launches": len(drain), "groups_per_launch": len(gbytes),
            "timing": "CUDA events around each engine launch on its stream, max over ranks",
            "largest_group": {"achieved": asym, "frac": asym / peak if asym else None,
                              "group_bytes": big_m.size_bytes, "us": big_m.time_sec * 1e6,
                              "from": "the largest size of this run's on-box calibration sweep (one group, "
                                      "idle engine, cold L2)"}})
        if N > 1:
            roof["frac_vs_770"] = achieved / NVLINK_PEER_GBS
        if 1 < N <= OTHER_PROTOCOL_MAX_N:
            # the same plan drained by the other protocol's engine (the
            # streamed one wins drains of many ready groups)
            alt = "stream" if engine_protocol == "chunked" else "chunked"
            comm.set_protocol(alt)
            p_alt = rt.Pipeline(dplans["mgwfbp"], trace, args.lr, args.algo, record_group_times=False,
                                l2_flush_bytes=flush, engine_ctas=args.engine_ctas)
            comm.set_protocol(args.protocol)
            D.barrier()
            d_alt = p_alt.drain(max(3, min(args.steps, 20)))
            p_alt.close()
            alt_s = D.max_over_ranks(statistics.mean(d_alt) / 1e3, dev)
            roof["other_protocol_drain"] = {"protocol": alt, "achieved": algo_bytes / alt_s / 1e9,
                                            "frac": algo_bytes / alt_s / 1e9 / peak,
                                            "launch_ms_mean": alt_s * 1e3}

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
        # the other protocol beside this run's (the calibration above): one
        # isolated group per size; the table reports both
        mine_proto = "chunked" if comm.protocol in ("auto", "chunked") else "stream"
        alt_proto = "stream" if mine_proto == "chunked" else "chunked"
        iso = [None] * len(big)
        if N <= OTHER_PROTOCOL_MAX_N:
            comm.set_protocol(alt_proto)
            mm = comm.calibrate_engine([m.size_bytes for m in big], warmup=2, reps=9, algo=args.algo,
                                       engine_ctas=args.engine_ctas if args.engine_ctas != 0 else -1,
                                       dtype=rt.BF16 if bf16 else rt.F32)
            comm.set_protocol(args.protocol)
            iso = [D.max_over_ranks(x.time_sec, dev) for x in mm]
        nv = [None] * len(big)
        if comm.nvls_ready:
            mm = comm.calibrate([m.size_bytes for m in big], warmup=2, reps=9, algo="nvls")
            nv = [D.max_over_ranks(x.time_sec, dev) for x in mm]
        for m, tn, tv, ti in zip(big, ncclt, nv, iso):
            f = 2 * (N - 1) / N * m.size_bytes / 1e9
            bus[str(m.size_bytes)] = {"mgwfbp": f / m.time_sec, "nccl": f / tn,
                                      "mgwfbp_frac_900": f / m.time_sec / NVLINK_GBS}
            if ti:
                bus[str(m.size_bytes)]["mgwfbp_" + mine_proto] = f / m.time_sec
                bus[str(m.size_bytes)]["mgwfbp_" + alt_proto] = f / ti
            if tv:
                bus[str(m.size_bytes)]["nvls_standalone"] = f / tv

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        tags = [int(t) for t in plans["mgwfbp"].tags]
        times = cpu_pipeline_sample(tr_json, tags, 1, args.lr, threads, args.cpu_budget_s)
        cpu = {"value": len(times) / sum(times), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{len(times)} iterations of the CPU Algorithm-2 restatement (oracle/mgw_oracle.c, "
                         f"same trace/plan, P=1, {threads} threads)"
                         + ("; the CPU path reduces fp32 gradients (no bf16 CPU pipeline)" if bf16 else ""),
               "detail": {"host": host_info(), "solver_1core": solver_table(),
                          "allreduce_sgd_config1_r50_2ranks": allreduce_cpu_config1()}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": (f"synthetic uniform[-1,1) {args.dtype} gradients"
                     + (" (fp32 accumulation, fp32 master weights)" if bf16 else "")
                     + "; backward replayed from B200-measured per-tensor t_b"),
            "config": cfg,
            "exposed_comm_ms": ms_step - cfg["compute_ms"],
            "iteration_bound": {"ms": bound_ms, "frac": bound_ms / ms_step,
                                "formula": "max(t_f + sum t_b, t_f + t_b[last layer] + sum_g 2(P-1)/P*S_g / 900 GB/s)"},
            "gpu": {"comm": ("persistent engine, %s CTAs" % ("1/SM" if args.engine_ctas < 0 else args.engine_ctas))
                            if args.engine_ctas else "one fused kernel launch per group",
                    "algo": args.algo, "tuning": comm.tuning(), "ipc_ranks_mapped": peers, "nvls": nvls,
                    "engine_protocol": engine_protocol,
                    "l2_flush": f"{args.l2_flush_mib} MiB streaming stores on the comm stream during the forward "
                                "replay, every iteration"},
            "calibration": {"plan_model": {"a_us": model.a * 1e6, "b_ps_per_byte": model.b * 1e12, "how": model_how},
                            "onbox": {"a_us": onbox_model.a * 1e6, "b_ps_per_byte": onbox_model.b * 1e12,
                                      "how": onbox_how, "sizes": len(meas), "largest_bytes": meas[-1].size_bytes,
                                      "largest_us": meas[-1].time_sec * 1e6,
                                      "plan_sha256": D.plan_digest(onbox_plan.tags)[:16],
                                      "groups": sum(1 for i, t in enumerate(onbox_plan.tags)
                                                    if i == 0 or int(t) == 0),
                                      "predicted_ms": gs.iteration_time(trace, onbox_plan,
                                                                        onbox_model).iteration_time * 1e3}},
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
