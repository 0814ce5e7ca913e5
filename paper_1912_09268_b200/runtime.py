"""Device runtime: communicator, device plans, fused merged all-reduce,
backward-replay pipeline and calibration — thin Python handles over the C
ABI (include/mgwfbp.h). PyTorch is used only as plumbing: device memory for
gradients/weights, the current CUDA stream, and torch.distributed to swap
the CUDA IPC handles once at start-up (paper Algorithm 2 line 8, Bcast).
"""
from __future__ import annotations

import ctypes as C
import weakref
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import arr
from .gradsched import (AllReduceModel, CommMeasurement, MergePlan, ModelTrace, check,
                        fit_model)

ALGO = {"auto": 0, "oneshot": 1, "twoshot": 2, "nvls": 3}
SGD = 1
WRITE_GRAD = 2


def _stream_ptr(stream) -> int:
    if isinstance(stream, int):
        return stream
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


F32, BF16 = 0, 1  # mgw_dtype (gradient / merge-arena element type)
PROTOCOLS = {"stream": 0, "chunked": 1, "auto": 2}  # MGW_PROTO_*


def padded_elems(counts: Sequence[int], dtype: int = F32) -> int:
    """Merge-layout size in elements: every layer starts on a 16-byte
    boundary (4 fp32 / 8 bf16 elements)."""
    g = 8 if dtype == BF16 else 4
    return sum((int(c) + g - 1) // g * g for c in counts)


def dtype_of(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(f"gradients must be float32 or bfloat16, got {t.dtype}")


class _Owner:
    """Native handles form a tree — communicator > device plans > pipelines /
    engines — and a child must be destroyed before its parent. close()
    closes the live children first, so teardown order never depends on the
    garbage collector (which finalises reference cycles in arbitrary order)."""

    def _adopt(self, child) -> None:
        if not hasattr(self, "_children"):
            self._children = weakref.WeakSet()
        self._children.add(child)

    def _close_children(self) -> None:
        kids = list(getattr(self, "_children", ()))
        if kids:
            self._children.clear()
        for child in kids:
            child.close()


class Comm(_Owner):
    """One rank's communicator (or a single-GPU loopback of `nranks` ranks)."""

    def __init__(self, rank: int, nranks: int, device: int, arena_bytes: int,
                 group=None, loopback: bool = False, exchange=None):
        """exchange: optional callable(bytes) -> list of every rank's bytes
        (rank order) used to swap the CUDA IPC handles instead of
        torch.distributed (e.g. a file rendezvous for profiler runs)."""
        self.rank, self.nranks, self.device = rank, nranks, device
        self.loopback = loopback
        h = C.c_void_p()
        if loopback:
            check(_lib.mgw_comm_create_loopback(nranks, device, arena_bytes, C.byref(h)))
        else:
            check(_lib.mgw_comm_create(rank, nranks, device, arena_bytes, C.byref(h)))
        self.handle = h
        if not loopback and nranks > 1:
            self._exchange(group, exchange)

    @classmethod
    def create_loopback(cls, nranks: int, device: int, arena_bytes: int) -> "Comm":
        return cls(0, nranks, device, arena_bytes, loopback=True)

    def _exchange(self, group, exchange=None) -> None:
        size = _lib.mgw_comm_handle_size()
        blob = (C.c_uint8 * size)()
        check(_lib.mgw_comm_export_handle(self.handle, blob))
        if exchange is not None:
            gathered = list(exchange(bytes(blob)))
        else:
            import torch.distributed as dist

            gathered: List[Optional[bytes]] = [None] * self.nranks
            dist.all_gather_object(gathered, bytes(blob), group=group)
        allb = b"".join(gathered)
        buf = (C.c_uint8 * len(allb)).from_buffer_copy(allb)
        check(_lib.mgw_comm_open_peers(self.handle, buf))

    def set_oneshot_max(self, nbytes: int) -> None:
        check(_lib.mgw_comm_set_oneshot_max(self.handle, int(nbytes)))

    def set_ll_max(self, nbytes: int) -> None:
        """One-shot groups up to nbytes travel as LL packets (0: never)."""
        check(_lib.mgw_comm_set_ll_max(self.handle, int(nbytes)))

    def set_small_tile_max(self, nbytes: int) -> None:
        """Groups below nbytes use 8 KiB tiles (more CTAs per group)."""
        check(_lib.mgw_comm_set_small_tile_max(self.handle, int(nbytes)))

    def set_chunk_tiles(self, max_tiles: int, min_chunks: int = 1) -> None:
        """Chunked protocol: a CTA's tiles run in pipelined chunks of <=
        max_tiles tiles and at least min_chunks chunks when it owns enough."""
        check(_lib.mgw_comm_set_chunk_tiles(self.handle, int(max_tiles), int(min_chunks)))

    def set_protocol(self, protocol: str) -> None:
        """'auto' (default: chunked at P > 1, the TMA-fed engine at P = 1),
        'stream' (per-tile delivery counts, no barrier after the entry
        barrier; pipelines launch their last-ready group chunked) or
        'chunked' (one cross-rank barrier per chunk)."""
        check(_lib.mgw_comm_set_protocol(self.handle, PROTOCOLS[protocol]))

    def set_stream_batches(self, credit_batch: int = 8, ag_batch: int = 4) -> None:
        """Streamed protocol publication batches (credit_batch in 1, 2, 4, 8)."""
        check(_lib.mgw_comm_set_stream_batches(self.handle, int(credit_batch), int(ag_batch)))

    @property
    def protocol(self) -> str:
        v = C.c_int()
        check(_lib.mgw_comm_get_protocol(self.handle, C.byref(v)))
        return {i: n for n, i in PROTOCOLS.items()}[v.value]

    def num_peers(self) -> int:
        """Ranks this communicator can address (itself included)."""
        v = C.c_int()
        check(_lib.mgw_comm_num_peers(self.handle, C.byref(v)))
        return v.value

    def failed(self) -> bool:
        """True once a kernel of this communicator gave up a bounded wait
        (host-mapped flag: no CUDA call, no sync)."""
        v = C.c_int()
        check(_lib.mgw_comm_error(self.handle, C.byref(v)))
        return bool(v.value)

    def nvls_supported(self) -> bool:
        """Multicast objects available (NVSwitch + fabric manager) and P > 1."""
        v = C.c_int()
        check(_lib.mgw_comm_nvls_supported(self.handle, C.byref(v)))
        return bool(v.value)

    def enable_nvls(self, min_bytes: int = 0, chunk_tiles: int = 4, group=None, exchange=None) -> None:
        """Collective: bind every rank's copy of one arena slot to a multicast
        object (rank 0 creates it, the peers import it; a barrier separates
        join and bind), then route fp32 groups of >= min_bytes through the
        switch-reduced path (0: only when asked with algo='nvls').
        exchange: optional callable(bytes) -> list of every rank's bytes, as
        for the IPC handles."""
        if exchange is None:
            import torch.distributed as dist

            def exchange(blob: bytes) -> List[bytes]:
                got: List[Optional[bytes]] = [None] * self.nranks
                dist.all_gather_object(got, blob, group=group)
                return got  # type: ignore[return-value]

        def phase(fn, payload=lambda: b"") -> List[bytes]:
            # every rank reports its outcome with the phase's payload, so a
            # failure on one rank raises on all of them (nobody is left
            # waiting in the next exchange)
            err = None
            try:
                fn()
            except Exception as e:  # noqa: BLE001 - re-raised below on every rank
                err = e
            got = list(exchange((b"1" if err is None else b"0") + payload()))
            if any(g[:1] != b"1" for g in got):
                raise RuntimeError(f"NVLS setup failed on rank(s) "
                                   f"{[r for r, g in enumerate(got) if g[:1] != b'1']}") from err
            return [g[1:] for g in got]

        size = _lib.mgw_nvls_handle_size()
        blob = (C.c_uint8 * size)()
        h0 = phase(lambda: check(_lib.mgw_comm_nvls_create(self.handle, blob)), lambda: bytes(blob))[0]
        phase(lambda: check(_lib.mgw_comm_nvls_join(self.handle, (C.c_uint8 * size).from_buffer_copy(h0))))
        phase(lambda: check(_lib.mgw_comm_nvls_bind(self.handle)))  # every GPU joined before anyone binds
        self.set_nvls(min_bytes, chunk_tiles)

    def set_nvls(self, min_bytes: int, chunk_tiles: int = 4) -> None:
        check(_lib.mgw_comm_set_nvls(self.handle, int(min_bytes), int(chunk_tiles)))

    @property
    def nvls_ready(self) -> bool:
        v = C.c_int()
        check(_lib.mgw_comm_nvls_ready(self.handle, C.byref(v)))
        return bool(v.value)

    def set_max_ctas(self, n: int) -> None:
        """Cap the CTAs of standalone fused launches (0: one per SM)."""
        check(_lib.mgw_comm_set_max_ctas(self.handle, int(n)))

    def tuning(self) -> dict:
        """The communicator's knob values."""
        o, l, t = C.c_uint64(), C.c_uint64(), C.c_uint64()
        ct, mc = C.c_uint32(), C.c_uint32()
        check(_lib.mgw_comm_get_tuning(self.handle, C.byref(o), C.byref(l), C.byref(t), C.byref(ct), C.byref(mc)))
        return {"oneshot_max": o.value, "ll_max": l.value, "small_tile_max": t.value,
                "chunk_tiles": ct.value, "min_chunks": mc.value, "protocol": self.protocol}

    @property
    def ll_max_bytes(self) -> int:
        return self.tuning()["ll_max"]

    @property
    def oneshot_max(self) -> int:
        v = C.c_uint64()
        check(_lib.mgw_comm_get_oneshot_max(self.handle, C.byref(v)))
        return v.value

    def allreduce_(self, buf: torch.Tensor, algo: str = "auto", stream=None) -> torch.Tensor:
        """In-place SUM all-reduce (rank order) of a contiguous fp32 tensor."""
        assert buf.dtype == torch.float32 and buf.is_cuda and buf.is_contiguous()
        check(_lib.mgw_allreduce(self.handle, buf.data_ptr(), buf.numel(), ALGO[algo], _stream_ptr(stream)))
        return buf

    def calibrate(self, sizes: Sequence[int], warmup: int = 3, reps: int = 20,
                  algo: str = "auto") -> List[CommMeasurement]:
        """N1: on-box fused all-reduce size sweep; median seconds per size."""
        out = (_lib.Meas * len(sizes))()
        check(_lib.mgw_calibrate(self.handle, arr(C.c_uint64, sizes), len(sizes), warmup, reps,
                                 ALGO[algo], out))
        return [CommMeasurement(out[i].size_bytes, out[i].time_sec) for i in range(len(sizes))]

    def calibrate_ce(self, sizes: Sequence[int], warmup: int = 3, reps: int = 15) -> List[CommMeasurement]:
        """Copy-engine pushes (rank -> rank+1 peer copy): median seconds per size."""
        out = (_lib.Meas * len(sizes))()
        check(_lib.mgw_calibrate_ce(self.handle, arr(C.c_uint64, sizes), len(sizes), warmup, reps, out))
        return [CommMeasurement(out[i].size_bytes, out[i].time_sec) for i in range(len(sizes))]

    def calibrate_engine(self, sizes: Sequence[int], warmup: int = 2, reps: int = 5,
                         algo: str = "auto", engine_ctas: int = -1, dtype: int = 0) -> List[CommMeasurement]:
        """N1 for engine pipelines: median per-group device time in the
        persistent comm engine (one group per iteration, ready at once);
        dtype: gradient type of the group (sizes in bytes)."""
        out = (_lib.Meas * len(sizes))()
        check(_lib.mgw_calibrate_engine_ex(self.handle, arr(C.c_uint64, sizes), len(sizes), warmup, reps,
                                           ALGO[algo], engine_ctas, int(dtype), out))
        return [CommMeasurement(out[i].size_bytes, out[i].time_sec) for i in range(len(sizes))]

    def close(self) -> None:
        self._close_children()
        if self.handle:
            check(_lib.mgw_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class DevicePlan(_Owner):
    """A merge plan bound to this rank's gradient / weight tensors.

    grads / weights: one CUDA tensor per layer in forward order (for a
    loopback comm: a list per emulated rank). Gradients are fp32 or bf16
    (all the same type); weights are fp32 master weights.
    """

    def __init__(self, comm: Comm, grads, weights, plan: MergePlan):
        self.comm = comm
        self.handle = None
        if comm.loopback:
            assert len(grads) == comm.nranks
            flat_g = [t for per in grads for t in per]
            flat_w = [t for per in weights for t in per] if weights is not None else None
            L = len(grads[0])
        else:
            flat_g, flat_w, L = list(grads), (list(weights) if weights is not None else None), len(grads)
        self.L = L
        self._keep = (flat_g, flat_w)  # tensors must outlive the plan
        counts = [int(t.numel()) for t in flat_g[:L]]
        self.counts = counts
        self.dtype = dtype_of(flat_g[0])
        if any(dtype_of(t) != self.dtype for t in flat_g):
            raise TypeError("all gradients of a plan must have the same dtype")
        if flat_w is not None and any(t.dtype != torch.float32 for t in flat_w):
            raise TypeError("weights must be float32 (master weights)")
        gp = arr(C.c_void_p, (t.data_ptr() for t in flat_g))
        wp = arr(C.c_void_p, (t.data_ptr() for t in flat_w)) if flat_w is not None else None
        h = C.c_void_p()
        check(_lib.mgw_plan_create_ex(comm.handle, L, gp, wp, arr(C.c_uint64, counts),
                                      arr(C.c_uint8, (int(t) for t in plan.tags)), self.dtype, C.byref(h)))
        self.handle = h
        comm._adopt(self)
        n = C.c_int()
        check(_lib.mgw_plan_num_groups(h, C.byref(n)))
        self.n_groups = n.value

    def group_span(self, g: int) -> Tuple[int, int, int]:
        b, c, by = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(_lib.mgw_plan_group_span(self.handle, g, C.byref(b), C.byref(c), C.byref(by)))
        return b.value, c.value, by.value

    def pack(self, g: int, scale: float, merge_buf: torch.Tensor, stream=None) -> None:
        check(_lib.mgw_pack(self.handle, g, scale, merge_buf.data_ptr(), _stream_ptr(stream)))

    def unpack_sgd(self, g: int, merge_buf: torch.Tensor, lr: float, write_grad: bool = False,
                   stream=None) -> None:
        check(_lib.mgw_unpack_sgd(self.handle, g, merge_buf.data_ptr(), lr, int(write_grad),
                                  _stream_ptr(stream)))

    def group_allreduce(self, g: int, lr: float, epilogue: int = SGD, algo: str = "auto",
                        stream=None) -> None:
        check(_lib.mgw_group_allreduce(self.handle, g, lr, epilogue, ALGO[algo], _stream_ptr(stream)))

    def close(self) -> None:
        self._close_children()
        if self.handle:
            check(_lib.mgw_plan_destroy(self.handle))
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class Pipeline:
    """Paper Algorithm 2 on one GPU: backward replay on a compute stream,
    each merge group's fused all-reduce on a comm stream the moment its head
    layer is ready, one CUDA graph per iteration."""

    def __init__(self, dplan: DevicePlan, trace: ModelTrace, lr: float, algo: str = "auto",
                 record_group_times: bool = False, l2_flush_bytes: int = 0, engine_ctas: int = -1,
                 h2d: Optional[Tuple[torch.Tensor, torch.Tensor]] = None,
                 d2h: Optional[Tuple[torch.Tensor, torch.Tensor]] = None):
        """engine_ctas: -1 persistent comm engine with one CTA per SM, > 0 that
        many CTAs, 0 = one fused kernel launch per group.
        h2d=(pinned_host_src, device_dst) / d2h=(pinned_host_dst, device_src):
        per-step host I/O captured into the iteration graph (end-to-end runs)."""
        self.dplan = dplan
        self.handle = None
        self.engine_ctas = engine_ctas
        self._io = (h2d, d2h)  # keep the buffers alive
        tb = arr(C.c_double, (l.backward_time for l in trace.layers))
        h = C.c_void_p()
        if h2d is None and d2h is None:
            check(_lib.mgw_pipeline_create(dplan.handle, tb, float(trace.forward_time), lr, ALGO[algo],
                                           int(record_group_times), int(l2_flush_bytes), int(engine_ctas),
                                           C.byref(h)))
        else:
            hs, hd = h2d if h2d is not None else (None, None)
            dd, ds = d2h if d2h is not None else (None, None)
            for t in (hs, dd):
                if t is not None and not t.is_pinned():
                    raise ValueError("host buffers of the step I/O must be pinned")
            nb_in = hs.numel() * hs.element_size() if hs is not None else 0
            nb_out = dd.numel() * dd.element_size() if dd is not None else 0
            check(_lib.mgw_pipeline_create_io(
                dplan.handle, tb, float(trace.forward_time), lr, ALGO[algo], int(record_group_times),
                int(l2_flush_bytes), int(engine_ctas),
                hs.data_ptr() if hs is not None else None, hd.data_ptr() if hd is not None else None, nb_in,
                dd.data_ptr() if dd is not None else None, ds.data_ptr() if ds is not None else None, nb_out,
                C.byref(h)))
        self.handle = h
        dplan._adopt(self)
        s = C.c_void_p()
        check(_lib.mgw_pipeline_stream(h, C.byref(s)))
        self.stream = torch.cuda.ExternalStream(s.value, device=torch.device("cuda", dplan.comm.device))

    def launch(self, iters: int = 1) -> None:
        check(_lib.mgw_pipeline_launch(self.handle, iters))

    def run(self, iters: int) -> List[float]:
        out = (C.c_float * iters)()
        check(_lib.mgw_pipeline_run(self.handle, iters, out))
        return list(out)

    def drain(self, iters: int) -> List[float]:
        """Standalone engine launches with every group ready (each after the
        pipeline's L2 flush): per-launch device ms of the whole plan's merged
        all-reduce + SGD — the kernel the roofline is quoted on."""
        out = (C.c_float * iters)()
        check(_lib.mgw_pipeline_drain(self.handle, iters, out))
        return list(out)

    def device_timeline(self) -> dict:
        """Last iteration on the device clock (engine pipelines with
        record_group_times): replay span, end of the last group's comm, and
        the exposed tail between them, in microseconds."""
        G = self.dplan.n_groups
        st = (C.c_uint64 * max(1, 2 * G))()
        check(_lib.mgw_pipeline_stamps(self.handle, st))
        eng = (C.c_uint32 * 4)()
        clk = (C.c_uint64 * 2)()
        check(_lib.mgw_pipeline_debug(self.handle, eng, clk))
        t0, rend = clk[0], clk[1]
        ends = [st[2 * g + 1] for g in range(G) if st[2 * g + 1]]
        end = max(ends) if ends else rend
        return {"replay_us": (rend - t0) / 1e3, "comm_end_us": (end - t0) / 1e3,
                "tail_us": (end - rend) / 1e3}

    @property
    def engine_protocol(self) -> str:
        """'stream' or 'chunked' for an engine pipeline ('none' without one)."""
        v = C.c_int()
        check(_lib.mgw_pipeline_streamed(self.handle, C.byref(v)))
        return "stream" if v.value else ("chunked" if self.engine_ctas != 0 else "none")

    def group_times_ms(self) -> List[float]:
        out = (C.c_float * max(1, self.dplan.n_groups))()
        check(_lib.mgw_pipeline_group_times(self.handle, out))
        return list(out)[: self.dplan.n_groups]

    def close(self) -> None:
        if self.handle:
            check(_lib.mgw_pipeline_destroy(self.handle))
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class CopyEngine:
    """Copy-engine mode of a real backward (mgw_ce_*): each group's gradients
    go to the peers' arenas as DMA copies when the group is marked ready (no
    SM taken from the backward); join() reduces every tile + SGD full width.
    The plan's gradients must be one flat buffer in the merge layout."""

    def __init__(self, dplan: DevicePlan, lr: float):
        self.dplan = dplan
        self.handle = None
        h = C.c_void_p()
        check(_lib.mgw_ce_create(dplan.handle, lr, C.byref(h)))
        self.handle = h
        dplan._adopt(self)

    def begin(self, stream=None) -> None:
        check(_lib.mgw_ce_begin(self.handle, _stream_ptr(stream)))

    def mark_ready(self, g: int, stream=None) -> None:
        check(_lib.mgw_ce_mark_ready(self.handle, g, _stream_ptr(stream)))

    def join(self, stream=None) -> None:
        check(_lib.mgw_ce_join(self.handle, _stream_ptr(stream)))

    @property
    def signals_without_sm(self) -> bool:
        """True: the delivery signals are stream memory operations (no SM), so
        fused tail launches may precede join() and overlap the reduce."""
        v = C.c_int()
        check(_lib.mgw_ce_signals_without_sm(self.handle, C.byref(v)))
        return bool(v.value)

    def set_tail(self, n_tail: int) -> None:
        """Leave groups [0, n_tail) to the caller (no copy, no reduce)."""
        check(_lib.mgw_ce_set_tail(self.handle, int(n_tail)))

    def check(self) -> None:
        check(_lib.mgw_ce_check(self.handle))

    def close(self) -> None:
        if self.handle:
            check(_lib.mgw_ce_destroy(self.handle))
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def kernel_launches() -> int:
    return int(_lib.mgw_kernel_launches())


def calibrated_model(comm: Comm, sizes: Sequence[int], warmup: int = 3, reps: int = 20,
                     algo: str = "auto") -> Tuple[AllReduceModel, List[CommMeasurement]]:
    meas = comm.calibrate(sizes, warmup, reps, algo)
    return fit_model(meas), meas
