"""The C ABI from a plain-C host (examples/mgw_c_host.c): it must compile
against include/mgwfbp.h + libmgwfbp.so (CPU), and run bit-exact (GPU)."""
import os
import subprocess

import pytest

from conftest import ROOT

CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
LIB = os.path.join(ROOT, "paper_1912_09268_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "mgw_c_host")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA, "include"),
           os.path.join(ROOT, "examples", "mgw_c_host.c"), "-o", exe, "-L" + LIB, "-lmgwfbp",
           "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-Wl,-rpath," + LIB,
           "-Wl,-rpath," + os.path.join(CUDA, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_host_compiles_against_the_c_abi(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_host_runs_bit_exact(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout
