"""API drop-in check: the reference's OWN Catch2 unit and acceptance suites
(/root/reference/proj/tests/*.cpp, compiled where they lie) build against
this repo's include/gradsched headers and pass when linked to libmgwfbp.so.

The Catch2 dependency (absent in this image) is replaced by our shim in
tests/cpp/catch_shim. test_cli.cpp is excluded: it drives the reference CLI
binary, which needs CLI11 (absent) and is out of scope.
Skipped where /root/reference does not exist (the GPU box).
"""
import os
import subprocess

import pytest

from conftest import REFERENCE, ROOT, has_reference

pytestmark = pytest.mark.skipif(not has_reference(), reason="/root/reference not present")

UNIT_FILES = ["test_comm_model.cpp", "test_trace.cpp", "test_timeline.cpp", "test_planner.cpp",
              "test_sweep.cpp"]


def _nlohmann():
    import glob

    for p in glob.glob("/opt/prime-rl/.venv/lib/python3.*/site-packages/include/cudnn_frontend/thirdparty"):
        if os.path.exists(os.path.join(p, "nlohmann", "json.hpp")):
            return p
    pytest.skip("nlohmann json not found")


def _build(tmp_path, sources, name, extra=()):
    lib_dir = os.path.join(ROOT, "paper_1912_09268_b200", "lib")
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", *extra,
           "-I", os.path.join(ROOT, "tests", "cpp", "catch_shim"), "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(REFERENCE, "tests"), "-I", _nlohmann(),
           f'-DGRADSCHED_FIXTURE_DIR="{REFERENCE}/tests/fixtures"', f'-DGRADSCHED_DATA_DIR="{REFERENCE}/data"']
    cmd += [os.path.join(REFERENCE, "tests", s) for s in sources]
    cmd += [os.path.join(ROOT, "tests", "cpp", "catch_shim", "catch_main.cpp"),
            "-L", lib_dir, "-lmgwfbp", f"-Wl,-rpath,{lib_dir}", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_reference_unit_suites_pass_against_our_headers(tmp_path):
    exe = _build(tmp_path, UNIT_FILES, "unit")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "48 test cases" in r.stdout and "0 failed" in r.stdout


def test_reference_cli_suite_passes_against_our_cli(tmp_path):
    """The reference's test_cli.cpp (15 cases: outputs byte-equal to the
    library exports, exit codes 0/2/3/4) driving OUR CLI binary."""
    cli = os.path.join(ROOT, "paper_1912_09268_b200", "bin", "gradsched")
    assert os.path.exists(cli), "build the CLI: make -C paper_1912_09268_b200/csrc"
    exe = _build(tmp_path, ["test_cli.cpp"], "cli_tests", extra=[f'-DGRADSCHED_CLI_PATH="{cli}"'])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "15 test cases" in r.stdout and "0 failed" in r.stdout


def test_reference_acceptance_suite_passes(tmp_path):
    exe = _build(tmp_path, ["acceptance_tests.cpp"], "acceptance")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    assert r.stdout.count("[PASS]") == 8 and "[FAIL]" not in r.stdout
