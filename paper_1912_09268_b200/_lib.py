"""ctypes binding of the C ABI in include/mgwfbp.h (libmgwfbp.so).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1912_09268_b200/csrc``). There is no fallback: if the shared
object is missing, importing this module raises, so nothing can silently run
a CPU path in place of the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmgwfbp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_1912_09268_b200/csrc`). There is no CPU fallback."
    )

lib = C.CDLL(LIB_PATH)

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p


class Meas(C.Structure):
    _fields_ = [("size_bytes", C.c_uint64), ("time_sec", C.c_double)]


def _proto(name, argtypes, restype=C.c_int):
    fn = getattr(lib, name)
    fn.argtypes = argtypes
    fn.restype = restype
    return fn


mgw_last_error = _proto("mgw_last_error", [], C.c_char_p)
mgw_last_error_kind = _proto("mgw_last_error_kind", [], C.c_char_p)
mgw_version = _proto("mgw_version", [], C.c_char_p)
mgw_fit = _proto("mgw_fit", [C.POINTER(Meas), C.c_size_t, f64p, f64p])
mgw_load_measurements_csv = _proto(
    "mgw_load_measurements_csv", [C.c_char_p, C.POINTER(Meas), C.c_size_t, C.POINTER(C.c_size_t)]
)
mgw_coefficients = _proto(
    "mgw_coefficients", [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, f64p, f64p]
)
mgw_load_trace = _proto(
    "mgw_load_trace",
    [C.c_char_p, C.POINTER(C.c_size_t), f64p, C.POINTER(C.c_int), u64p, f64p, C.c_size_t],
)
_plan_args = [u64p, f64p, C.c_size_t, C.c_double, C.c_int, C.c_double, C.c_double]
mgw_plan_optimal = _proto("mgw_plan_optimal", _plan_args + [u8p])
mgw_plan_greedy = _proto("mgw_plan_greedy", _plan_args + [u8p])
mgw_plan_brute_force = _proto("mgw_plan_brute_force", _plan_args + [C.c_size_t, u8p, f64p])
mgw_predict = _proto("mgw_predict", _plan_args + [u8p, f64p, f64p, f64p, f64p, f64p])
_table_args = [u64p, f64p, C.c_size_t, C.c_double, C.c_int, C.POINTER(Meas), C.c_size_t]
mgw_plan_optimal_table = _proto("mgw_plan_optimal_table", _table_args + [u8p])
mgw_predict_table = _proto("mgw_predict_table", _table_args + [u8p, f64p])
mgw_baseline_times = _proto("mgw_baseline_times", _plan_args + [f64p, f64p])
mgw_synth_trace_json = _proto(
    "mgw_synth_trace_json",
    [C.c_size_t, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_char_p,
     C.c_size_t],
    C.c_long,
)

mgw_comm_create = _proto("mgw_comm_create", [C.c_int, C.c_int, C.c_int, C.c_size_t, C.POINTER(vp)])
mgw_comm_create_loopback = _proto(
    "mgw_comm_create_loopback", [C.c_int, C.c_int, C.c_size_t, C.POINTER(vp)]
)
mgw_comm_handle_size = _proto("mgw_comm_handle_size", [], C.c_size_t)
mgw_comm_export_handle = _proto("mgw_comm_export_handle", [vp, vp])
mgw_comm_open_peers = _proto("mgw_comm_open_peers", [vp, vp])
mgw_comm_destroy = _proto("mgw_comm_destroy", [vp])
mgw_comm_num_peers = _proto("mgw_comm_num_peers", [vp, C.POINTER(C.c_int)])
mgw_comm_set_oneshot_max = _proto("mgw_comm_set_oneshot_max", [vp, C.c_uint64])
mgw_comm_get_oneshot_max = _proto("mgw_comm_get_oneshot_max", [vp, u64p])
mgw_comm_set_max_ctas = _proto("mgw_comm_set_max_ctas", [vp, C.c_int])
mgw_comm_set_ll_max = _proto("mgw_comm_set_ll_max", [vp, C.c_uint64])
mgw_comm_set_small_tile_max = _proto("mgw_comm_set_small_tile_max", [vp, C.c_uint64])
mgw_comm_set_chunk_tiles = _proto("mgw_comm_set_chunk_tiles", [vp, C.c_uint32, C.c_uint32])
mgw_comm_set_protocol = _proto("mgw_comm_set_protocol", [vp, C.c_int])
mgw_pipeline_streamed = _proto("mgw_pipeline_streamed", [vp, C.POINTER(C.c_int)])
mgw_comm_set_stream_batches = _proto("mgw_comm_set_stream_batches", [vp, C.c_uint32, C.c_uint32])
mgw_comm_get_protocol = _proto("mgw_comm_get_protocol", [vp, C.POINTER(C.c_int)])
mgw_comm_error = _proto("mgw_comm_error", [vp, C.POINTER(C.c_int)])
mgw_nvls_handle_size = _proto("mgw_nvls_handle_size", [], C.c_size_t)
mgw_comm_nvls_supported = _proto("mgw_comm_nvls_supported", [vp, C.POINTER(C.c_int)])
mgw_comm_nvls_create = _proto("mgw_comm_nvls_create", [vp, vp])
mgw_comm_nvls_join = _proto("mgw_comm_nvls_join", [vp, vp])
mgw_comm_nvls_bind = _proto("mgw_comm_nvls_bind", [vp])
mgw_comm_nvls_ready = _proto("mgw_comm_nvls_ready", [vp, C.POINTER(C.c_int)])
mgw_comm_set_nvls = _proto("mgw_comm_set_nvls", [vp, C.c_uint64, C.c_uint32])
mgw_comm_set_nvls_skip = _proto("mgw_comm_set_nvls_skip", [vp, C.c_uint32])
mgw_comm_get_tuning = _proto("mgw_comm_get_tuning", [vp, u64p, u64p, u64p, C.POINTER(C.c_uint32),
                                                      C.POINTER(C.c_uint32)])
mgw_plan_create = _proto(
    "mgw_plan_create", [vp, C.c_size_t, C.POINTER(vp), C.POINTER(vp), u64p, u8p, C.POINTER(vp)]
)
mgw_plan_create_ex = _proto(
    "mgw_plan_create_ex", [vp, C.c_size_t, C.POINTER(vp), C.POINTER(vp), u64p, u8p, C.c_int, C.POINTER(vp)]
)
mgw_plan_destroy = _proto("mgw_plan_destroy", [vp])
mgw_plan_num_groups = _proto("mgw_plan_num_groups", [vp, C.POINTER(C.c_int)])
mgw_plan_group_span = _proto("mgw_plan_group_span", [vp, C.c_int, u64p, u64p, u64p])
mgw_pack = _proto("mgw_pack", [vp, C.c_int, C.c_float, vp, vp])
mgw_unpack_sgd = _proto("mgw_unpack_sgd", [vp, C.c_int, vp, C.c_float, C.c_int, vp])
mgw_group_allreduce = _proto("mgw_group_allreduce", [vp, C.c_int, C.c_float, C.c_int, C.c_int, vp])
mgw_allreduce = _proto("mgw_allreduce", [vp, vp, C.c_size_t, C.c_int, vp])
mgw_calibrate = _proto(
    "mgw_calibrate", [vp, u64p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.POINTER(Meas)]
)
mgw_pipeline_create = _proto(
    "mgw_pipeline_create",
    [vp, f64p, C.c_double, C.c_float, C.c_int, C.c_int, C.c_size_t, C.c_int, C.POINTER(vp)],
)
mgw_calibrate_engine = _proto(
    "mgw_calibrate_engine",
    [vp, u64p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Meas)],
)
mgw_calibrate_engine_ex = _proto(
    "mgw_calibrate_engine_ex",
    [vp, u64p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Meas)],
)
mgw_pipeline_create_io = _proto(
    "mgw_pipeline_create_io",
    [vp, f64p, C.c_double, C.c_float, C.c_int, C.c_int, C.c_size_t, C.c_int, vp, vp, C.c_size_t, vp, vp,
     C.c_size_t, C.POINTER(vp)],
)
mgw_pipeline_destroy = _proto("mgw_pipeline_destroy", [vp])
mgw_pipeline_launch = _proto("mgw_pipeline_launch", [vp, C.c_int])
mgw_pipeline_run = _proto("mgw_pipeline_run", [vp, C.c_int, f32p])
mgw_pipeline_group_times = _proto("mgw_pipeline_group_times", [vp, f32p])
mgw_pipeline_stream = _proto("mgw_pipeline_stream", [vp, C.POINTER(vp)])
mgw_pipeline_debug = _proto("mgw_pipeline_debug", [vp, C.POINTER(C.c_uint32), u64p])
mgw_pipeline_stamps = _proto("mgw_pipeline_stamps", [vp, u64p])
mgw_pipeline_stamps_raw = _proto("mgw_pipeline_stamps_raw", [vp, u64p, C.c_size_t, C.POINTER(C.c_size_t)])
mgw_pipeline_drain = _proto("mgw_pipeline_drain", [vp, C.c_int, f32p])
mgw_engine_create = _proto("mgw_engine_create", [vp, C.c_float, C.c_int, C.c_int, C.c_int, C.POINTER(vp)])
mgw_engine_begin = _proto("mgw_engine_begin", [vp, vp])
mgw_engine_mark_ready = _proto("mgw_engine_mark_ready", [vp, C.c_int, vp])
mgw_engine_join = _proto("mgw_engine_join", [vp, vp])
mgw_engine_set_tail = _proto("mgw_engine_set_tail", [vp, C.c_int])
mgw_engine_check = _proto("mgw_engine_check", [vp])
mgw_ce_create = _proto("mgw_ce_create", [vp, C.c_float, C.POINTER(vp)])
mgw_ce_begin = _proto("mgw_ce_begin", [vp, vp])
mgw_ce_mark_ready = _proto("mgw_ce_mark_ready", [vp, C.c_int, vp])
mgw_ce_join = _proto("mgw_ce_join", [vp, vp])
mgw_ce_set_tail = _proto("mgw_ce_set_tail", [vp, C.c_int])
mgw_ce_signals_without_sm = _proto("mgw_ce_signals_without_sm", [vp, C.POINTER(C.c_int)])
mgw_ce_check = _proto("mgw_ce_check", [vp])
mgw_ce_destroy = _proto("mgw_ce_destroy", [vp])
mgw_calibrate_ce = _proto("mgw_calibrate_ce", [vp, u64p, C.c_size_t, C.c_int, C.c_int, C.POINTER(Meas)])
mgw_kernel_launches = _proto("mgw_kernel_launches", [], C.c_uint64)

# Every symbol the header declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    name
    for name in dir()
    if name.startswith("mgw_") and callable(globals()[name])
]


def arr(ctype, values):
    """A ctypes array holding `values`."""
    values = list(values)
    return (ctype * max(1, len(values)))(*values)
