"""CPU checks of the boundary and the reduction oracle (no GPU compute):
  * libmgwfbp.so loads and exports every symbol include/*.h declares;
  * the C-ABI status/exception mapping mirrors the reference classes;
  * the oracle's pack / rank-order reduction / SGD agrees with an
    independent numpy float32 statement of the same semantics.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import pyoracle
from paper_1912_09268_b200 import _lib
from paper_1912_09268_b200 import gradsched as gs


def _declared_symbols():
    syms = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            syms |= set(re.findall(r"\b(mgw_[a-z0-9_]+)\s*\(", text))
    return syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 35
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert declared <= set(_lib.EXPORTED), sorted(declared - set(_lib.EXPORTED))


def test_version_and_error_kind():
    assert b"sm_100a" in _lib.mgw_version()
    with pytest.raises(gs.ParseError, match="cannot open"):
        gs.load_trace("/nonexistent/trace.json")
    with pytest.raises(gs.ParseError, match="header"):
        p = os.path.join(ROOT, "tests", "golden", "three_layer.json")
        gs.load_measurements_csv(p)


def test_device_api_without_gpu_fails_loudly_not_silently():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by -m gpu tests")
    h = ctypes.c_void_p()
    rc = _lib.mgw_comm_create(0, 1, 0, 1 << 20, ctypes.byref(h))
    assert rc == 6  # MGW_ERR_CUDA: no device, no CPU fallback
    assert _lib.mgw_last_error_kind() == b"CudaError"


def test_merge_offsets_are_16_byte_aligned():
    counts = [7, 0, 1, 4, 4097, 3]
    offs = pyoracle.merge_offsets(counts)
    assert offs == [0, 8, 8, 12, 16, 4116, 4120]
    assert all(o % 4 == 0 for o in offs)


def _np_reduce(grads, weights, lr, P):
    s = np.float32(1.0 / P)
    out_w, out_g = [], []
    for l in range(len(grads[0])):
        acc = (grads[0][l] * s).astype(np.float32)
        for r in range(1, P):
            acc = (acc + (grads[r][l] * s).astype(np.float32)).astype(np.float32)
        step = (np.float32(lr) * acc).astype(np.float32)
        out_w.append([(weights[r][l] - step).astype(np.float32) for r in range(P)])
        out_g.append(acc)
    return out_w, out_g


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_oracle_reduction_matches_numpy_rank_order(P):
    rng = np.random.default_rng(P)
    counts = [0, 1, 7, 4096, 5000, 33]
    grads = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    weights = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    want_w, want_g = _np_reduce(grads, weights, 0.01, P)
    pyoracle.allreduce_sgd(grads, weights, [0, 1, 0, 1, 1, 0], 0.01, write_grad=True)
    for l in range(len(counts)):
        for r in range(P):
            assert np.array_equal(weights[r][l], want_w[l][r])
            assert np.array_equal(grads[r][l], want_g[l])


@pytest.mark.parametrize("P", [2, 4, 8])
def test_oracle_nvls_variant_is_the_exact_sum_rounded_once(P):
    """NVLS numerics (the NVSwitch's multimem.ld_reduce, measured on B200 by
    tools/nvls_probe.cu): the exact sum of the P scaled fp32 values, rounded
    once to fp32 — checked against rational arithmetic; at P = 2 it is the
    rank-order sum bit for bit."""
    from fractions import Fraction

    rng = np.random.default_rng(100 + P)
    counts = [0, 1, 7, 300, 33]
    grads = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    weights = [[rng.uniform(-1, 1, c).astype(np.float32) for c in counts] for _ in range(P)]
    s = np.float32(1.0 / P)
    exact = [np.array([float(sum(Fraction(float(grads[r][l][j] * s)) for r in range(P)))
                       for j in range(counts[l])], dtype=np.float64).astype(np.float32) for l in range(len(counts))]
    want_w = [[(weights[r][l] - np.float32(0.01) * exact[l]).astype(np.float32) for l in range(len(counts))]
              for r in range(P)]
    g_rank = [[g.copy() for g in per] for per in grads]
    w_rank = [[w.copy() for w in per] for per in weights]
    pyoracle.allreduce_sgd(g_rank, w_rank, [0, 1, 0, 1, 0], 0.01, write_grad=True)
    pyoracle.allreduce_sgd_nvls(grads, weights, [0, 1, 0, 1, 0], 0.01, write_grad=True)
    for l in range(len(counts)):
        for r in range(P):
            assert np.array_equal(grads[r][l], exact[l])
            assert np.array_equal(weights[r][l], want_w[r][l])
            if P == 2:
                assert np.array_equal(grads[r][l], g_rank[r][l])
                assert np.array_equal(weights[r][l], w_rank[r][l])


def test_oracle_pack_layout():
    rng = np.random.default_rng(7)
    grads = [rng.uniform(-1, 1, c).astype(np.float32) for c in (5, 0, 9)]
    out = pyoracle.pack(grads, 0, 3, 0.5)
    assert out.size == 8 + 0 + 12
    assert np.array_equal(out[:5], (grads[0] * np.float32(0.5)).astype(np.float32))
    assert np.all(out[5:8] == 0)
    assert np.array_equal(out[8:17], (grads[2] * np.float32(0.5)).astype(np.float32))
    assert np.all(out[17:] == 0)


def test_cpu_pipeline_runs_and_respects_replay_time():
    counts = [1000, 2000, 0, 500]
    t_b = [2e-3, 1e-3, 1e-3, 1e-3]
    grads = [[np.ones(c, np.float32) for c in counts]]
    weights = [[np.zeros(c, np.float32) for c in counts]]
    times = pyoracle.pipeline_run(grads, weights, counts, t_b, 1e-3, [0, 1, 0, 0], 0.5, 2, 3)
    assert len(times) == 3
    assert all(t >= 6e-3 for t in times)  # t_f + sum(t_b) replayed
    # 3 iterations of w -= 0.5 * 1 (P=1)
    assert np.all(weights[0][0] == -1.5)


def test_oracle_bf16_rounding_is_round_to_nearest_even():
    """The bf16 oracle's fp32 -> bf16 rounding (C and its numpy restatement)
    against torch's conversion, on random values and on exact ties."""
    import torch

    rng = np.random.default_rng(7)
    x = rng.standard_normal(200000).astype(np.float32) * np.float32(1e3)
    # exact ties: bf16 value + half an ulp, both parities of the kept bit
    base = (rng.integers(0x0080, 0x7F00, 5000, dtype=np.uint32) << 16) | 0x8000
    ties = base.view(np.float32)
    x = np.concatenate([x, ties, -ties, np.float32([0.0, -0.0, 1e-40, -1e-40, 3.4e38])]).astype(np.float32)
    want = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = pyoracle.f32_to_bf16(x)
    assert np.array_equal(got, want)
    c = np.array([pyoracle.ORC.orc_f32_to_bf16(float(v)) for v in x[-6000:]], dtype=np.uint16)
    assert np.array_equal(c, want[-6000:])
    assert np.array_equal(pyoracle.bf16_to_f32(got), torch.from_numpy(want.view(np.int16)).view(torch.bfloat16).float().numpy())


def test_oracle_bf16_allreduce_semantics():
    """One rank-order bf16 reduction restated by hand on a tiny case."""
    g = [[np.array([0x3F80, 0x4000, 0xC040], dtype=np.uint16)],   # 1, 2, -3
         [np.array([0x3F80, 0x3F00, 0x4040], dtype=np.uint16)]]   # 1, 0.5, 3
    w = [[np.zeros(3, dtype=np.float32)], [np.ones(3, dtype=np.float32)]]
    pyoracle.allreduce_sgd_bf16(g, w, [0], 0.5, write_grad=True)
    red = np.float32([1.0, 1.25, 0.0])
    assert np.array_equal(pyoracle.bf16_to_f32(g[0][0]), red) and np.array_equal(g[0][0], g[1][0])
    assert np.array_equal(w[0][0], -np.float32(0.5) * red) and np.array_equal(w[1][0], 1 - np.float32(0.5) * red)


def test_bf16_merge_layout_pads_layers_to_16_bytes():
    """bf16 plans pad every layer to 8 elements (16 bytes): the Python
    mirror, the oracle and the TMA / LL granule agree."""
    from paper_1912_09268_b200 import runtime as rt

    counts = [1, 7, 8, 9, 0, 4097, 3]
    offs = pyoracle.merge_offsets_granule(counts, 8)
    assert all(o % 8 == 0 for o in offs)
    assert offs[-1] == rt.padded_elems(counts, rt.BF16)
    assert pyoracle.merge_offsets(counts)[-1] == rt.padded_elems(counts, rt.F32)


def test_scaling_projection_runs_on_committed_calibrations():
    """§8f row 3: the measured-coefficient projection (ring alpha/beta fitted
    to the on-box N=2,4 calibrations, then the reference sweep via the CLI)."""
    import subprocess
    import sys

    calib = os.path.join(ROOT, "profiles", "calib")
    if not os.path.exists(os.path.join(calib, "calib_resnet50_P2.csv")):
        pytest.skip("no committed calibrations")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "project_scaling.py"), "resnet50", calib,
                          "2,4,8,64"], capture_output=True, text=True, check=True).stdout
    rows = [l.split() for l in out.splitlines() if l and not l.startswith("#") and l.split()[0].isdigit()]
    eff = {(int(r[0]), r[1]): float(r[5]) for r in rows}
    assert eff[(64, "mgwfbp")] >= eff[(64, "wfbp")]  # merging never loses under the reference model
    assert 0 < eff[(8, "mgwfbp")] <= 1.0
