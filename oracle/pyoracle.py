"""ctypes handles on the oracle libraries. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.

  C    = oracle/_build/libmgw_oracle.so   (CPU restatement, mgw_oracle.c)
  REF  = oracle/_ref/libgradsched_ref.so  (the reference headers compiled in
                                           place; None when never built)
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_PATH = os.path.join(HERE, "_build", "libmgw_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libgradsched_ref.so")

u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
fpp = C.POINTER(C.c_void_p)


def _load(path: str) -> Optional[C.CDLL]:
    return C.CDLL(path) if os.path.exists(path) else None


ORC = _load(C_PATH)
REF = _load(REF_PATH)

_P = [u64p, f64p, C.c_size_t, C.c_double, C.c_int, C.c_double, C.c_double]

if ORC is not None:
    ORC.orc_optimal_plan.argtypes = _P + [u8p]
    ORC.orc_greedy_plan.argtypes = _P + [u8p]
    ORC.orc_iteration_time.argtypes = _P + [u8p]
    ORC.orc_iteration_time.restype = C.c_double
    ORC.orc_fit.argtypes = [u64p, f64p, C.c_size_t, f64p, f64p]
    ORC.orc_merge_offsets.argtypes = [u64p, C.c_size_t, u64p]
    ORC.orc_merge_offsets.restype = None
    ORC.orc_pack.argtypes = [fpp, u64p, u64p, C.c_size_t, C.c_size_t, C.c_float, C.c_void_p]
    ORC.orc_pack.restype = None
    ORC.orc_allreduce_sgd.argtypes = [C.c_int, fpp, fpp, u64p, C.c_size_t, u8p, C.c_float, C.c_int]
    ORC.orc_allreduce_sgd_nvls.argtypes = [C.c_int, fpp, fpp, u64p, C.c_size_t, u8p, C.c_float, C.c_int]
    ORC.orc_allreduce_sgd.restype = None
    ORC.orc_pipeline_run.argtypes = [C.c_int, fpp, fpp, u64p, f64p, C.c_size_t, C.c_double, u8p,
                                     C.c_float, C.c_int, C.c_int, f64p]
    ORC.orc_f32_to_bf16.argtypes = [C.c_float]
    ORC.orc_f32_to_bf16.restype = C.c_uint16
    ORC.orc_bf16_to_f32.argtypes = [C.c_uint16]
    ORC.orc_bf16_to_f32.restype = C.c_float
    ORC.orc_merge_offsets_granule.argtypes = [u64p, C.c_size_t, C.c_uint64, u64p]
    ORC.orc_merge_offsets_granule.restype = None
    ORC.orc_pack_bf16.argtypes = [fpp, u64p, u64p, C.c_size_t, C.c_size_t, C.c_float, C.c_void_p]
    ORC.orc_pack_bf16.restype = None
    ORC.orc_allreduce_sgd_bf16.argtypes = [C.c_int, fpp, fpp, u64p, C.c_size_t, u8p, C.c_float, C.c_int]
    ORC.orc_allreduce_sgd_bf16.restype = None

if REF is not None:
    REF.ref_optimal_plan.argtypes = _P + [u8p]
    REF.ref_greedy_plan.argtypes = _P + [u8p]
    REF.ref_brute_force_plan.argtypes = _P + [u8p, f64p]
    REF.ref_iteration_time.argtypes = _P + [u8p, f64p, f64p]
    REF.ref_synceasgd_time.argtypes = _P + [f64p]
    REF.ref_fit.argtypes = [u64p, f64p, C.c_size_t, f64p, f64p]
    REF.ref_fit_csv.argtypes = [C.c_char_p, f64p, f64p]
    REF.ref_synth_trace.argtypes = [C.c_size_t, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                    C.c_int, C.c_uint64, C.c_char_p, C.c_size_t]
    REF.ref_synth_trace.restype = C.c_long


def _arrs(params: Sequence[int], t_b: Sequence[float]):
    L = len(params)
    return (C.c_uint64 * L)(*[int(p) for p in params]), (C.c_double * L)(*[float(t) for t in t_b]), L


def _plan(lib, fn: str, params, t_b, t_f, bpe, a, b) -> Optional[List[int]]:
    p, tb, L = _arrs(params, t_b)
    out = (C.c_uint8 * L)()
    rc = getattr(lib, fn)(p, tb, L, float(t_f), int(bpe), float(a), float(b), out)
    return list(out) if rc == 0 else None


def orc_optimal(params, t_b, t_f, bpe, a, b):
    return _plan(ORC, "orc_optimal_plan", params, t_b, t_f, bpe, a, b)


def orc_greedy(params, t_b, t_f, bpe, a, b):
    return _plan(ORC, "orc_greedy_plan", params, t_b, t_f, bpe, a, b)


def ref_optimal(params, t_b, t_f, bpe, a, b):
    return _plan(REF, "ref_optimal_plan", params, t_b, t_f, bpe, a, b)


def ref_greedy(params, t_b, t_f, bpe, a, b):
    return _plan(REF, "ref_greedy_plan", params, t_b, t_f, bpe, a, b)


def orc_iteration_time(params, t_b, t_f, bpe, a, b, tags) -> float:
    p, tb, L = _arrs(params, t_b)
    return ORC.orc_iteration_time(p, tb, L, float(t_f), int(bpe), float(a), float(b),
                                  (C.c_uint8 * L)(*tags))


def ref_iteration_time(params, t_b, t_f, bpe, a, b, tags) -> float:
    p, tb, L = _arrs(params, t_b)
    it, no = C.c_double(), C.c_double()
    rc = REF.ref_iteration_time(p, tb, L, float(t_f), int(bpe), float(a), float(b),
                                (C.c_uint8 * L)(*tags), C.byref(it), C.byref(no))
    assert rc == 0
    return it.value


def orc_fit(sizes, times):
    n = len(sizes)
    a, b = C.c_double(), C.c_double()
    rc = ORC.orc_fit((C.c_uint64 * n)(*sizes), (C.c_double * n)(*times), n, C.byref(a), C.byref(b))
    return (a.value, b.value) if rc == 0 else None


def ref_fit(sizes, times):
    n = len(sizes)
    a, b = C.c_double(), C.c_double()
    rc = REF.ref_fit((C.c_uint64 * n)(*sizes), (C.c_double * n)(*times), n, C.byref(a), C.byref(b))
    return (a.value, b.value) if rc == 0 else None


def merge_offsets(counts: Sequence[int]) -> List[int]:
    L = len(counts)
    out = (C.c_uint64 * (L + 1))()
    ORC.orc_merge_offsets((C.c_uint64 * L)(*counts), L, out)
    return list(out)


def _ptrs(arrays: Sequence[np.ndarray]):
    return (C.c_void_p * len(arrays))(*[a.ctypes.data if a is not None else None for a in arrays])


def pack(grads: Sequence[np.ndarray], first: int, last: int, scale: float) -> np.ndarray:
    counts = [g.size for g in grads]
    offs = merge_offsets(counts)
    out = np.zeros(offs[last] - offs[first], dtype=np.float32)
    ORC.orc_pack(_ptrs(grads), (C.c_uint64 * len(counts))(*counts),
                 (C.c_uint64 * len(offs))(*offs), first, last, scale, out.ctypes.data)
    return out


def allreduce_sgd(grads: List[List[np.ndarray]], weights: List[List[np.ndarray]], tags, lr: float,
                  write_grad: bool = False) -> None:
    """In place on the numpy arrays: grads[r][l], weights[r][l]."""
    P, L = len(grads), len(grads[0])
    counts = [g.size for g in grads[0]]
    ORC.orc_allreduce_sgd(P, _ptrs([g for per in grads for g in per]),
                          _ptrs([w for per in weights for w in per]),
                          (C.c_uint64 * L)(*counts), L, (C.c_uint8 * L)(*tags), lr, int(write_grad))


def allreduce_sgd_nvls(grads: List[List[np.ndarray]], weights: List[List[np.ndarray]], tags, lr: float,
                       write_grad: bool = False) -> None:
    """allreduce_sgd with the NVLS numerics: each element's sum is the exact
    sum of the P scaled values rounded once to fp32."""
    P, L = len(grads), len(grads[0])
    counts = [g.size for g in grads[0]]
    ORC.orc_allreduce_sgd_nvls(P, _ptrs([g for per in grads for g in per]),
                               _ptrs([w for per in weights for w in per]),
                               (C.c_uint64 * L)(*counts), L, (C.c_uint8 * L)(*tags), lr, int(write_grad))


# ---- bf16 gradients -----------------------------------

def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits (uint16), round to nearest even: the vectorised
    restatement of orc_f32_to_bf16 (tests check it against the C oracle and
    against torch's conversion)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def bf16_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(h, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def merge_offsets_granule(counts: Sequence[int], granule: int) -> List[int]:
    L = len(counts)
    out = (C.c_uint64 * (L + 1))()
    ORC.orc_merge_offsets_granule((C.c_uint64 * L)(*counts), L, granule, out)
    return list(out)


def pack_bf16(grads: Sequence[np.ndarray], first: int, last: int, scale: float) -> np.ndarray:
    """grads: uint16 (bf16 bits) arrays; returns the uint16 merge buffer."""
    counts = [g.size for g in grads]
    offs = merge_offsets_granule(counts, 8)
    out = np.zeros(offs[last] - offs[first], dtype=np.uint16)
    ORC.orc_pack_bf16(_ptrs(grads), (C.c_uint64 * len(counts))(*counts),
                      (C.c_uint64 * len(offs))(*offs), first, last, scale, out.ctypes.data)
    return out


def allreduce_sgd_bf16(grads: List[List[np.ndarray]], weights: List[List[np.ndarray]], tags, lr: float,
                       write_grad: bool = False) -> None:
    """In place: grads[r][l] uint16 (bf16 bits), weights[r][l] float32."""
    P, L = len(grads), len(grads[0])
    counts = [g.size for g in grads[0]]
    ORC.orc_allreduce_sgd_bf16(P, _ptrs([g for per in grads for g in per]),
                               _ptrs([w for per in weights for w in per]),
                               (C.c_uint64 * L)(*counts), L, (C.c_uint8 * L)(*tags), lr, int(write_grad))


def pipeline_run(grads, weights, counts, t_b, t_f, tags, lr, threads, iters) -> List[float]:
    P, L = len(grads), len(counts)
    out = (C.c_double * max(1, iters))()
    rc = ORC.orc_pipeline_run(P, _ptrs([g for per in grads for g in per]),
                              _ptrs([w for per in weights for w in per]),
                              (C.c_uint64 * L)(*counts), (C.c_double * L)(*t_b), L, float(t_f),
                              (C.c_uint8 * L)(*tags), lr, threads, iters, out)
    assert rc == 0
    return list(out)[:iters]
