"""The bench's roofline kernel standalone (tools only; ncu target): the
persistent engine draining a whole trace's optimal plan with every group
ready at launch (mgw_pipeline_drain), on one GPU — P = 1, or P emulated
ranks in loopback (engine grid (ctas, P)). No replay kernel runs beside it,
so ncu can serialise and replay the launch.

usage: python tools/drain_probe.py --trace bert_large [--P 1] [--iters 3]
  ncu --set full -k regex:engine_kernel --launch-count 1 python tools/drain_probe.py ...
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", default="bert_large")
    ap.add_argument("--P", type=int, default=1)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--flush-mib", type=int, default=256)
    ap.add_argument("--stamps", action="store_true", help="per-group device stamps of the last drain")
    args = ap.parse_args()
    tr = gs.load_trace(os.path.join(ROOT, "traces", f"{args.trace}.json"))
    calib = os.path.join(ROOT, "profiles", "calib", f"calib_{args.trace}_P{args.P}.csv")
    plan = gs.optimal_plan(tr, gs.fit_model(gs.load_measurements_csv(calib)))
    counts = [l.params for l in tr.layers]
    P = args.P
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    grads = [[torch.empty(c, device="cuda").uniform_(-1, 1, generator=gen) for c in counts] for _ in range(P)]
    weights = [[torch.empty(c, device="cuda").uniform_(-1, 1, generator=gen) for c in counts] for _ in range(P)]
    if P == 1:
        comm = rt.Comm(0, 1, 0, 4 * rt.padded_elems(counts))
        dp = rt.DevicePlan(comm, grads[0], weights[0], plan)
    else:
        comm = rt.Comm.create_loopback(P, 0, 4 * rt.padded_elems(counts))
        dp = rt.DevicePlan(comm, grads, weights, plan)
    pipe = rt.Pipeline(dp, tr, 0.01, l2_flush_bytes=args.flush_mib << 20, engine_ctas=-1,
                       record_group_times=args.stamps)
    ms = pipe.drain(args.iters)
    if args.stamps:
        import ctypes as C

        from paper_1912_09268_b200 import _lib

        G = dp.n_groups
        st = (C.c_uint64 * (2 * G))()
        gs.check(_lib.mgw_pipeline_stamps(pipe.handle, st))
        t0 = min(st[2 * g] for g in range(G) if st[2 * g])
        rows = [((st[2 * g] - t0) / 1e3, (st[2 * g + 1] - t0) / 1e3, dp.group_span(g)[2]) for g in range(G)]
        for g in list(range(G - 1, G - 12, -1)) + list(range(min(10, G) - 1, -1, -1)):
            print(f"group {g:4d} bytes {rows[g][2]:10d} start {rows[g][0]:8.2f} us end {rows[g][1]:8.2f} us")
        print("span us", max(r[1] for r in rows), "sum of group durations us", sum(r[1] - r[0] for r in rows))
        cap = G * 4096 * 2
        raw = (C.c_uint64 * cap)()
        cols = C.c_size_t()
        gs.check(_lib.mgw_pipeline_stamps_raw(pipe.handle, raw, cap, C.byref(cols)))
        nc = cols.value
        # the CTA that ran the FIFO-last group: its own timeline
        for cta in sorted({c for g in range(G) for c in range(nc) if raw[(g * nc + c) * 2]}, key=lambda c: -max(
                (raw[(g * nc + c) * 2 + 1] for g in range(G) if raw[(g * nc + c) * 2]), default=0))[:2]:
            seq = sorted((raw[(g * nc + cta) * 2] - t0, raw[(g * nc + cta) * 2 + 1] - t0, g) for g in range(G)
                         if raw[(g * nc + cta) * 2])
            print(f"CTA {cta}: " + "  ".join(f"g{g}[{a / 1e3:.2f}-{b / 1e3:.2f}]" for a, b, g in seq))
    S = sum(dp.group_span(g)[2] for g in range(dp.n_groups))
    hbm = 3 * S * P
    print(json.dumps({"trace": args.trace, "P": P, "groups": dp.n_groups, "grad_bytes_per_rank": S,
                      "launch_ms": ms, "median_ms": statistics.median(ms),
                      "hbm_algorithmic_bytes_per_launch": hbm,
                      "hbm_gbs": hbm / (statistics.median(ms) / 1e3) / 1e9, "tuning": comm.tuning()}), flush=True)
    pipe.close()
    dp.close()
    comm.close()


if __name__ == "__main__":
    main()
