"""Python mirror of the reference `gradsched` API, backed by libmgwfbp.so.

Same names, argument meaning and error classes as the reference C++ headers
(/root/reference/proj/include/gradsched/*.hpp) so that host code and tests
read like the reference's own:

    trace = load_trace("traces/resnet50.json")
    model = fit_model(measurements)                # comm_model.hpp:209
    plan  = optimal_plan(trace, model)             # planner.hpp:63
    tl    = iteration_time(trace, plan, model)     # timeline.hpp:158

Every numeric result comes from the C++ library through the C ABI
(include/mgwfbp.h); nothing here re-implements the arithmetic.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

from . import _lib
from ._lib import arr, lib


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """Base of all gradsched errors (reference errors.hpp:24-27)."""


class ValidationError(Error):
    pass


class ParseError(Error):
    pass


class FitError(Error):
    pass


class PlannerError(Error):
    pass


class GuardError(Error):
    pass


class CudaError(Error):
    """A CUDA runtime failure inside libmgwfbp (not in the reference)."""


_KINDS = {
    "ValidationError": ValidationError,
    "ParseError": ParseError,
    "FitError": FitError,
    "PlannerError": PlannerError,
    "GuardError": GuardError,
    "CudaError": CudaError,
}


def check(status: int) -> None:
    """Raise the reference-named exception for a non-zero mgw_status."""
    if status == 0:
        return
    msg = _lib.mgw_last_error().decode(errors="replace")
    kind = _lib.mgw_last_error_kind().decode()
    raise _KINDS.get(kind, Error)(msg)


# ------------------------------------------------------------- data model
@dataclass
class LayerProfile:
    """reference trace.hpp:38-42 (backward_time in seconds)."""

    name: str
    params: int
    backward_time: float


@dataclass
class ModelTrace:
    """reference trace.hpp:47-94; layers in forward order."""

    layers: List[LayerProfile] = field(default_factory=list)
    forward_time: float = 0.0
    bytes_per_element: int = 4

    def n_layers(self) -> int:
        return len(self.layers)

    def total_params(self) -> int:
        return sum(l.params for l in self.layers)

    # C-ABI marshalling
    def _c(self):
        L = len(self.layers)
        return (
            arr(C.c_uint64, (l.params for l in self.layers)),
            arr(C.c_double, (l.backward_time for l in self.layers)),
            L,
            float(self.forward_time),
            int(self.bytes_per_element),
        )


@dataclass
class AllReduceModel:
    """T(M) = a + b*M (reference comm_model.hpp:33-47)."""

    a: float = 0.0
    b: float = 0.0


@dataclass
class CommMeasurement:
    size_bytes: int
    time_sec: float


class LayerTag(enum.IntEnum):
    kNormal = 0
    kMerged = 1


@dataclass
class MergePlan:
    """reference timeline.hpp:36-67."""

    tags: List[LayerTag]

    @staticmethod
    def all_normal(n: int) -> "MergePlan":
        return MergePlan([LayerTag.kNormal] * n)

    @staticmethod
    def all_merged(n: int) -> "MergePlan":
        return MergePlan([LayerTag.kNormal] + [LayerTag.kMerged] * (n - 1)) if n else MergePlan([])

    def merged_count(self) -> int:
        return sum(1 for t in self.tags if t == LayerTag.kMerged)

    def groups(self) -> List[List[int]]:
        """0-based layer indices per group, ascending (apply_merge order)."""
        out: List[List[int]] = []
        for i, t in enumerate(self.tags):
            if i == 0 or t == LayerTag.kNormal:
                out.append([i])
            else:
                out[-1].append(i)
        return out

    def tag_bytes(self) -> bytes:
        return bytes(int(t) for t in self.tags)


@dataclass
class Timeline:
    """reference timeline.hpp:86-95 (the fields the C ABI returns)."""

    tau_b: List[float]
    tau_c: List[float]
    t_c: List[float]
    iteration_time: float
    comm_nonoverlap: float


@dataclass
class PlanSearchResult:
    plan: MergePlan
    iteration_time: float


class AllReduceAlgorithm(enum.IntEnum):
    kBinaryTree = 0
    kRecursiveDoubling = 1
    kRecursiveHalvingDoubling = 2
    kDoubleBinaryTrees = 3
    kRing = 4


@dataclass
class NetworkParams:
    alpha: float = 0.0
    beta: float = 0.0
    gamma: float = 0.0
    n_workers: int = 0


# --------------------------------------------------------------- functions
def coefficients_for(algo: AllReduceAlgorithm, net: NetworkParams, dbt_literal: bool = False) -> AllReduceModel:
    a, b = C.c_double(), C.c_double()
    check(_lib.mgw_coefficients(int(algo), net.alpha, net.beta, net.gamma, net.n_workers,
                                int(dbt_literal), C.byref(a), C.byref(b)))
    return AllReduceModel(a.value, b.value)


def allreduce_cost(model: AllReduceModel, size_bytes: float) -> float:
    """a + b*M evaluated by the C++ library's rule (no FMA)."""
    if not size_bytes >= 0.0:
        raise ValidationError("allreduce_cost: size_bytes must be >= 0")
    # Python floats are IEEE doubles; a + b*M here rounds identically to the
    # -ffp-contract=off C++ (two roundings).
    return model.a + model.b * size_bytes


def fit_model(samples: Sequence[CommMeasurement]) -> AllReduceModel:
    c = arr(_lib.Meas, (_lib.Meas(int(s.size_bytes), float(s.time_sec)) for s in samples))
    a, b = C.c_double(), C.c_double()
    check(_lib.mgw_fit(c, len(samples), C.byref(a), C.byref(b)))
    return AllReduceModel(a.value, b.value)


def load_measurements_csv(path: str) -> List[CommMeasurement]:
    n = C.c_size_t()
    check(_lib.mgw_load_measurements_csv(path.encode(), None, 0, C.byref(n)))
    buf = (_lib.Meas * max(1, n.value))()
    check(_lib.mgw_load_measurements_csv(path.encode(), buf, n.value, C.byref(n)))
    return [CommMeasurement(buf[i].size_bytes, buf[i].time_sec) for i in range(n.value)]


def load_trace(path: str) -> ModelTrace:
    """reference trace.hpp:148-219 (C++ parser; µs -> s)."""
    L = C.c_size_t()
    tf = C.c_double()
    bpe = C.c_int()
    check(_lib.mgw_load_trace(path.encode(), C.byref(L), C.byref(tf), C.byref(bpe), None, None, 0))
    params = (C.c_uint64 * L.value)()
    tb = (C.c_double * L.value)()
    check(_lib.mgw_load_trace(path.encode(), C.byref(L), C.byref(tf), C.byref(bpe), params, tb, L.value))
    with open(path) as f:
        names = [l["name"] for l in json.load(f)["layers"]]
    return ModelTrace(
        [LayerProfile(names[i], int(params[i]), float(tb[i])) for i in range(L.value)],
        tf.value,
        bpe.value,
    )


def _tags_from(buf, L) -> MergePlan:
    return MergePlan([LayerTag(buf[i]) for i in range(L)])


def optimal_plan(trace: ModelTrace, model: AllReduceModel) -> MergePlan:
    p, tb, L, tf, bpe = trace._c()
    out = (C.c_uint8 * max(1, L))()
    check(_lib.mgw_plan_optimal(p, tb, L, tf, bpe, model.a, model.b, out))
    return _tags_from(out, L)


def greedy_plan(trace: ModelTrace, model: AllReduceModel) -> MergePlan:
    p, tb, L, tf, bpe = trace._c()
    out = (C.c_uint8 * max(1, L))()
    check(_lib.mgw_plan_greedy(p, tb, L, tf, bpe, model.a, model.b, out))
    return _tags_from(out, L)


def brute_force_plan(trace: ModelTrace, model: AllReduceModel, max_layers: int = 20) -> PlanSearchResult:
    p, tb, L, tf, bpe = trace._c()
    out = (C.c_uint8 * max(1, L))()
    it = C.c_double()
    check(_lib.mgw_plan_brute_force(p, tb, L, tf, bpe, model.a, model.b, max_layers, out, C.byref(it)))
    return PlanSearchResult(_tags_from(out, L), it.value)


def iteration_time(trace: ModelTrace, plan: MergePlan, model: AllReduceModel) -> Timeline:
    p, tb, L, tf, bpe = trace._c()
    tags = arr(C.c_uint8, (int(t) for t in plan.tags))
    it, no = C.c_double(), C.c_double()
    tau_b, tau_c, t_c = ((C.c_double * max(1, L))() for _ in range(3))
    check(_lib.mgw_predict(p, tb, L, tf, bpe, model.a, model.b, tags, C.byref(it), C.byref(no),
                           tau_b, tau_c, t_c))
    return Timeline(list(tau_b)[:L], list(tau_c)[:L], list(t_c)[:L], it.value, no.value)


def _meas_arr(meas: Sequence[CommMeasurement]):
    out = (_lib.Meas * max(1, len(meas)))()
    for i, m in enumerate(meas):
        out[i].size_bytes, out[i].time_sec = int(m.size_bytes), float(m.time_sec)
    return out


def optimal_plan_table(trace: ModelTrace, meas: Sequence[CommMeasurement]) -> MergePlan:
    """B200 extension: optimal_plan's exact DP with T(M) interpolated from the
    measured calibration instead of a + b*M (mgw_plan_optimal_table)."""
    p, tb, L, tf, bpe = trace._c()
    out = (C.c_uint8 * max(1, L))()
    check(_lib.mgw_plan_optimal_table(p, tb, L, tf, bpe, _meas_arr(meas), len(meas), out))
    return _tags_from(out, L)


def iteration_time_table(trace: ModelTrace, plan: MergePlan, meas: Sequence[CommMeasurement]) -> float:
    """The serialised FIFO iteration time with the interpolated measured cost."""
    p, tb, L, tf, bpe = trace._c()
    tags = arr(C.c_uint8, (int(t) for t in plan.tags))
    it = C.c_double()
    check(_lib.mgw_predict_table(p, tb, L, tf, bpe, _meas_arr(meas), len(meas), tags, C.byref(it)))
    return it.value


def synceasgd_time(trace: ModelTrace, model: AllReduceModel) -> float:
    p, tb, L, tf, bpe = trace._c()
    s, n = C.c_double(), C.c_double()
    check(_lib.mgw_baseline_times(p, tb, L, tf, bpe, model.a, model.b, C.byref(s), C.byref(n)))
    return s.value


def naive_time(trace: ModelTrace, model: AllReduceModel) -> float:
    p, tb, L, tf, bpe = trace._c()
    s, n = C.c_double(), C.c_double()
    check(_lib.mgw_baseline_times(p, tb, L, tf, bpe, model.a, model.b, C.byref(s), C.byref(n)))
    return n.value


def speedup(n_workers: int, forward_time: float, backward_time: float, comm_nonoverlap: float) -> float:
    """N / (1 + r), r = comm_nonoverlap / (t_f + t_b) (reference timeline.hpp:225-233)."""
    compute = forward_time + backward_time
    if not compute > 0.0:
        raise ValidationError("speedup: forward + backward time must be > 0")
    return float(n_workers) / (1.0 + comm_nonoverlap / compute)


@dataclass
class SynthSpec:
    """reference trace.hpp:257-265."""

    n_layers: int = 0
    total_params: int = 0
    total_backward_time: float = 0.0
    forward_time: float = 0.0
    size_skew: float = 8.0
    bytes_per_element: int = 4
    seed: int = 0


def synth_trace_json(spec: SynthSpec) -> str:
    """Canonical save_trace() text of synth_trace(spec) (byte-stable)."""
    args = (spec.n_layers, spec.total_params, spec.total_backward_time, spec.forward_time,
            spec.size_skew, spec.bytes_per_element, spec.seed)
    n = _lib.mgw_synth_trace_json(*args, None, 0)
    if n < 0:
        check(-n)
    buf = C.create_string_buffer(n + 1)
    _lib.mgw_synth_trace_json(*args, buf, n + 1)
    return buf.value.decode()


def trace_from_arrays(params: Iterable[int], t_b: Iterable[float], t_f: float, bpe: int = 4,
                      names: Optional[Sequence[str]] = None) -> ModelTrace:
    params = list(params)
    t_b = list(t_b)
    names = list(names) if names is not None else [f"layer_{i + 1:03d}" for i in range(len(params))]
    return ModelTrace([LayerProfile(n, int(p), float(t)) for n, p, t in zip(names, params, t_b)], t_f, bpe)
