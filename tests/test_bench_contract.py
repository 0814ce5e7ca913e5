"""bench.py's contract on CPU: the reference arm prints one JSON line with
the contract's keys, never loads this package (its libmgwfbp.so), and both
arms build the identical `config` (same plan, same plan_sha256) from the
committed calibration — the GPU arm through the package's bit-exact
planner, the reference arm through the reference's own fit_model +
optimal_plan (oracle/_ref)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_reference

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_default_workload_is_the_largest_single_gpu_config():
    sys_argv = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = bench.parse_args()
    finally:
        sys.argv = sys_argv
    assert a.trace == "bert_large" and a.gpus == 1 and a.plan_source == "committed"


def test_reference_arm_prints_one_contract_line_without_the_package():
    code = (
        "import sys, os; sys.argv=['bench.py','--impl','reference','--steps','2','--warmup','3','--trace','googlenet'];"
        "sys.path.insert(0, os.getcwd()); import bench; rc = bench.main();"
        "maps = open('/proc/self/maps').read();"
        "print('PKG_LOADED', 'paper_1912_09268_b200' in sys.modules, 'libmgwfbp' in maps)"
    )
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "PKG_LOADED False False" in r.stdout, r.stdout[-500:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "exposed_comm_ms"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["workload"] == "googlenet" and d["unit"] == "worker-iters/s"
    assert d["config"]["calibration_csv"] == "profiles/calib/calib_googlenet_P1.csv"
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("trace", ["bert_large", "resnet50", "googlenet", "resnet152", "densenet201",
                                   "inception_v4"])
def test_both_arms_build_the_identical_config(trace, N):
    if not has_reference():
        pytest.skip("oracle/_ref needs the reference sources")
    from paper_1912_09268_b200 import gradsched as gs

    calib = bench.committed_calibration(trace, N)
    assert calib is not None, (trace, N)
    # GPU arm: the package's load_trace / fit_model / optimal_plan
    t = gs.load_trace(bench.trace_path(trace))
    plan = gs.optimal_plan(t, gs.fit_model(gs.load_measurements_csv(os.path.join(ROOT, calib))))
    tr = bench.load_trace_json(bench.trace_path(trace))
    gpu_cfg = bench.common_config(trace, tr, N, [int(x) for x in plan.tags], calib, 1.0, "fp32")
    # reference arm: the unmodified reference headers (oracle/_ref)
    a, b, kind = bench.ref_fit(os.path.join(ROOT, calib))
    tags, pkind = bench.ref_plan(tr, a, b, 4)
    assert kind == "reference" and pkind == "reference"
    ref_cfg = bench.common_config(trace, tr, N, tags, calib, 1.0, "fp32")
    assert gpu_cfg == ref_cfg
    # the parsed doubles equal the library's ModelTrace bit for bit
    assert tr["t_f"] == t.forward_time and tr["t_b"] == [l.backward_time for l in t.layers]
