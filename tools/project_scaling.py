"""Measured-coefficient scaling projection (tools only).

The on-box calibrations of the fused all-reduce at N = 2 and 4
(gpurun_out/calib_<trace>_P<N>.csv, written by bench.py) are fitted per N to
T(M) = a_N + b_N M (fit_model, reference comm_model.hpp:209-251), then to the
ring alpha-beta form of the reference's Table 2 (coefficients_for,
comm_model.hpp:140-191): a_N = 2(N-1) alpha, b_N = 2(N-1)/N beta (least
squares through the origin). The reference's own sweep (run_sweep,
sweep.hpp:92-173, via this repo's `gradsched sweep` CLI) then projects
naive / WFBP / SyncEASGD / MG-WFBP iteration time and speedup to N beyond
the box. The per-N measured rows use the planner with the measured (a_N,
b_N) directly.

usage: python tools/project_scaling.py TRACE [CALIB_DIR] [WORKERS]
"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402

trace_name = sys.argv[1]
calib_dir = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
workers = sys.argv[3] if len(sys.argv) > 3 else "2,4,8,16,32,64,72,128"
trace_path = os.path.join(ROOT, "traces", f"{trace_name}.json")
trace = gs.load_trace(trace_path)

fits = {}
for n in (2, 4, 8):
    p = os.path.join(calib_dir, f"calib_{trace_name}_P{n}.csv")
    if os.path.exists(p):
        fits[n] = gs.fit_model(gs.load_measurements_csv(p))
if len(fits) < 1:
    sys.exit(f"no calibration CSVs for {trace_name} in {calib_dir}")
alpha = sum(f.a * 2 * (n - 1) for n, f in fits.items()) / sum((2 * (n - 1)) ** 2 for n in fits)
beta = sum(f.b * 2 * (n - 1) / n for n, f in fits.items()) / sum((2 * (n - 1) / n) ** 2 for n in fits)

print(f"# trace {trace_name}: {len(trace.layers)} layers, t_f + sum t_b = "
      f"{(trace.forward_time + sum(l.backward_time for l in trace.layers)) * 1e3:.3f} ms (B200-measured)")
for n, f in sorted(fits.items()):
    t_mg = gs.iteration_time(trace, gs.optimal_plan(trace, f), f).iteration_time
    t_wf = gs.iteration_time(trace, gs.MergePlan.all_normal(len(trace.layers)), f).iteration_time
    t_sb = gs.naive_time(trace, f)
    print(f"# measured N={n}: a={f.a * 1e6:.2f} us  b={f.b * 1e12:.3f} ps/B  ->  predicted iter "
          f"MG-WFBP {t_mg * 1e3:.3f} / WFBP {t_wf * 1e3:.3f} / single-buffer {t_sb * 1e3:.3f} ms")
print(f"# ring fit over N={sorted(fits)}: alpha = {alpha * 1e6:.3f} us, beta = {beta * 1e12:.4f} ps/B "
      f"(a_N = 2(N-1) alpha, b_N = 2(N-1)/N beta)")
cli = os.path.join(ROOT, "paper_1912_09268_b200", "bin", "gradsched")
out = subprocess.run([cli, "sweep", trace_path, "--algo", "ring", "--alpha", repr(alpha), "--beta", repr(beta),
                      "--workers", workers], capture_output=True, text=True, check=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
print(f"{'N':>5s} {'strategy':>10s} {'iter_ms':>10s} {'nonoverlap_ms':>14s} {'speedup':>8s} {'eff':>6s} {'merged':>6s}")
for r in rows:
    n = int(r["n_workers"])
    sp = float(r["speedup"])
    print(f"{n:5d} {r['strategy']:>10s} {float(r['iter_time_us']) / 1e3:10.3f} "
          f"{float(r['comm_nonoverlap_us']) / 1e3:14.3f} {sp:8.2f} {sp / n:6.3f} {r['n_merged']:>6s}")
