"""MG-WFBP for a real PyTorch backward (paper Algorithm 2,
PAPER.md:486-563, and its system design PAPER.md:545-563).

The paper's C++ daemon thread pops layer ids from a queue the backward pushes
to and all-reduces each merged group when its last layer arrives. Here:

* the "queue" is a per-group ready flag on the GPU: an autograd
  post-accumulate-grad hook on every parameter counts the group's finished
  members and, when the group is complete, enqueues a 1-thread mark kernel
  on the current (compute) stream — no host synchronisation, no GIL wait;
* the "daemon thread" is the persistent comm engine kernel (launched at the
  start of the backward on its own stream, a few SMs): it reduces the groups
  FIFO in backward order over NVLink, fused with the SGD update
  `W = W - lr * mean(grad)` (paper line 15 of Algorithm 2);
* gradients live in one flat buffer with 16-byte aligned per-parameter
  views (`p.grad`), so autograd accumulates in place at stable addresses.

    sync = MGWFBP(model, comm, lr=0.01, plan=plan)
    for x, y in data:
        sync.begin()                 # zero grads, launch the engine
        loss_fn(model(x), y).backward()
        sync.end()                   # next forward waits for the SGD
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, List, Optional

import torch

from . import _lib
from .gradsched import MergePlan, check
from .runtime import ALGO, Comm, CopyEngine, DevicePlan, padded_elems


class MGWFBP:
    def __init__(self, model: torch.nn.Module, comm: Comm, lr: float, plan: Optional[MergePlan] = None,
                 algo: str = "auto", engine_ctas: int = 8, record_group_times: bool = False,
                 params: Optional[List[torch.nn.Parameter]] = None, tail_groups: int = 1,
                 mode: str = "auto", launch_ctas: int = 16):
        """params: the layer order of the plan / trace (forward order; the
        backward visits it last to first). Default: model.parameters().
        tail_groups: the last groups the backward makes ready (groups
        0..tail_groups-1) are reduced after the backward by a full-width
        fused kernel instead of the few-CTA engine — the SMs are free then.
        mode: "engine" — the persistent comm engine (engine_ctas CTAs for the
        whole backward); "launch" — one fused launch per group on a comm
        stream the moment the group is complete (launch_ctas CTAs, SMs held
        only while a group is in flight); "auto" — "ce" at P > 1, else
        "engine"; "ce" — copy-engine mode: each
        finished group's gradients go to the peers' arenas as DMA copies (no
        SM taken from the backward), one full-width reduce + SGD after it
        (runtime.CopyEngine; P > 1)."""
        if mode == "auto":  # measured fastest: copy engines at P > 1
            mode = "ce" if comm.nranks > 1 else "engine"
        if mode not in ("engine", "launch", "ce"):
            raise ValueError("mode must be 'auto', 'engine', 'launch' or 'ce'")
        self.mode, self.launch_ctas, self.comm = mode, int(launch_ctas), comm
        self.params: List[torch.nn.Parameter] = (list(params) if params is not None else
                                                 [p for p in model.parameters() if p.requires_grad])
        for p in self.params:
            if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
                raise ValueError("MGWFBP needs contiguous fp32 CUDA parameters")
        L = len(self.params)
        self.plan = plan if plan is not None else MergePlan.all_normal(L)
        if len(self.plan.tags) != L:
            raise ValueError(f"plan has {len(self.plan.tags)} tags for {L} parameters")
        counts = [p.numel() for p in self.params]
        dev = self.params[0].device
        self.flat_grad = torch.zeros(max(1, padded_elems(counts)), dtype=torch.float32, device=dev)
        off = 0
        grads = []
        for p, c in zip(self.params, counts):
            view = self.flat_grad[off:off + c]
            p.grad = view.view_as(p)
            grads.append(view)
            off += (c + 3) & ~3
        weights = [p.data.view(-1) for p in self.params]
        self.dplan = DevicePlan(comm, grads, weights, self.plan)
        self.lr, self.algo = lr, algo
        self.groups = self.plan.groups()
        self.handle = None
        self.ce = None
        if mode == "ce":
            self.ce = CopyEngine(self.dplan, lr)
            self.tail = max(0, min(int(tail_groups), len(self.groups) - 1))
            self.ce.set_tail(self.tail)
            self._ce_overlap = self.ce.signals_without_sm
        else:
            h = C.c_void_p()
            check(_lib.mgw_engine_create(self.dplan.handle, lr, ALGO[algo], engine_ctas,
                                         int(record_group_times), C.byref(h)))
            self.handle = h
            self.dplan._adopt(self)
            self.tail = max(0, min(int(tail_groups), len(self.groups)))
            check(_lib.mgw_engine_set_tail(h, self.tail))
        self.group_of = [0] * L
        for g, members in enumerate(self.groups):
            for i in members:
                self.group_of[i] = g
        self.remaining = [len(m) for m in self.groups]
        self._next = len(self.groups) - 1
        self._iters = 0
        self._launched = False
        self._lazy_launch = False
        self._hooks = [p.register_post_accumulate_grad_hook(self._hook(i)) for i, p in enumerate(self.params)]
        if mode == "launch":
            self.comm_stream = torch.cuda.Stream(device=dev)
            self._events = [torch.cuda.Event() for _ in range(len(self.groups) + 1)]

    def _launch(self, g: int, stream) -> None:
        """launch mode: group g on the comm stream after the work queued on `stream`."""
        ev = self._events[g]
        ev.record(torch.cuda.ExternalStream(stream) if isinstance(stream, int) else stream)
        self.comm_stream.wait_event(ev)
        self.comm.set_max_ctas(self.launch_ctas)
        check(_lib.mgw_group_allreduce(self.dplan.handle, g, self.lr, 1, ALGO[self.algo],
                                       self.comm_stream.cuda_stream))

    def _advance(self, stream) -> None:
        """launch mode: launch the complete groups in backward (FIFO) order.

        A group is launched only after every group before it in backward
        order: if parameter use differs between ranks (data-dependent unused
        parameters), hooks fire in different orders, but every rank still
        issues the same sequence of collective launches — the cross-rank
        barriers pair launches by order, not by group id."""
        while self._next >= self.tail and self.remaining[self._next] == 0:
            self._launch(self._next, stream)
            self._next -= 1

    def _hook(self, i: int):
        def hook(_p):
            g = self.group_of[i]
            self.remaining[g] -= 1
            if self.remaining[g] == 0 and self.mode == "ce":
                if g >= self.tail:  # a ring append, no CUDA call (the daemon records the event)
                    if self._ce_mark(self.ce.handle, g, self._ce_stream) != 0:
                        check(-1)
            elif self.remaining[g] == 0 and g >= self.tail and self.mode == "launch":
                self._advance(torch.cuda.current_stream())
            elif self.remaining[g] == 0 and g >= self.tail:
                stream = torch.cuda.current_stream().cuda_stream
                if self._lazy_launch and not self._launched:
                    # start the engine with the first finished group: the
                    # forward pass keeps every SM. Ordered after the compute
                    # stream's queued work — in particular the previous
                    # iteration's full-width tail launches, whose CTAs must
                    # all be resident (an engine holding SMs while waiting
                    # for marks queued behind them would deadlock).
                    check(_lib.mgw_engine_begin(self.handle, stream))
                    self._launched = True
                check(_lib.mgw_engine_mark_ready(self.handle, g, stream))
        return hook

    def begin(self) -> None:
        """Zero the gradients and start this iteration's comm engine.

        The first iteration runs the engine only after the backward: CUDA 12
        loads modules lazily at a kernel's first launch and that load waits
        for the context to go idle, so a backward launching kernels for the
        first time would stall behind the spinning engine (measured). After
        one iteration every kernel is loaded and the engine overlaps.
        (CUDA_MODULE_LOADING=EAGER removes the issue from the start.)"""
        for p in self.params:
            if p.grad is None or p.grad.data_ptr() < self.flat_grad.data_ptr():
                raise RuntimeError("a parameter's .grad was replaced; keep zero_grad(set_to_none=False)")
        self.flat_grad.zero_()
        self.remaining = [len(m) for m in self.groups]
        self._next = len(self.groups) - 1
        self._launched = False
        # overlap from the 2nd iteration (or from the start with eager module
        # loading); the engine starts at the first finished group
        self._lazy_launch = self._iters > 0 or os.environ.get("CUDA_MODULE_LOADING", "") == "EAGER"
        if self.mode == "ce":
            self._ce_stream = torch.cuda.current_stream().cuda_stream
            self._ce_mark = _lib.mgw_ce_mark_ready
            self.ce.begin(self._ce_stream)

    def end(self) -> None:
        """Make the current stream wait until every group's SGD is applied."""
        stream = torch.cuda.current_stream().cuda_stream
        missing = [g for g, r in enumerate(self.remaining) if r != 0 and g >= self.tail]
        if self.mode == "ce":
            for g in missing:  # parameters that got no gradient this iteration
                self.ce.mark_ready(g, torch.cuda.current_stream())
            # With a signal KERNEL the copy-engine reduce must come first, THEN
            # the tail groups' fused launches: a fused launch pairs its CTAs with
            # the peers' and may hold every SM while it waits, so it must never
            # run ahead of a peer's signal kernel (deadlock: rank r's reduce
            # spins for rank q's signal while rank q's SMs are held by its tail
            # kernel waiting for rank r's tail CTAs, measured at N = 4). With
            # stream-memop signals (no SM) the tail overlaps the reduce.
            overlap = self._ce_overlap  # SM-free signals: the tail may overlap the reduce
            if not overlap:
                self.ce.join(torch.cuda.current_stream())
            for g in reversed(range(self.tail)):
                check(_lib.mgw_group_allreduce(self.dplan.handle, g, self.lr, 1, ALGO[self.algo], stream))
            if overlap:
                self.ce.join(torch.cuda.current_stream())
        elif self.mode == "launch":
            for g in range(self._next, self.tail - 1, -1):  # the rest in order (incl. groups without gradients)
                self._launch(g, torch.cuda.current_stream())
            self._next = self.tail - 1
            done = self._events[-1]
            done.record(self.comm_stream)
            torch.cuda.current_stream().wait_event(done)
            self.comm.set_max_ctas(0)
        else:
            for g in missing:  # parameters that got no gradient this iteration
                check(_lib.mgw_engine_mark_ready(self.handle, g, stream))
            if not self._launched:
                check(_lib.mgw_engine_begin(self.handle, stream))
            check(_lib.mgw_engine_join(self.handle, stream))
        if self.mode != "ce":
            for g in reversed(range(self.tail)):  # backward order, full width
                check(_lib.mgw_group_allreduce(self.dplan.handle, g, self.lr, 1, ALGO[self.algo], stream))
        self._iters += 1
        # a timed-out wait of an earlier iteration (host-mapped flag: no sync);
        # its kernels skipped their SGD, so the weights are stale, not corrupt
        if self.comm.failed():
            raise RuntimeError("MG-WFBP: a cross-rank or ready wait timed out (a peer or a group never "
                               "arrived); the communicator has failed")

    def check(self) -> None:
        if self.ce is not None:
            self.ce.check()
        else:
            check(_lib.mgw_engine_check(self.handle))

    def group_times_ms(self) -> List[float]:
        out = (C.c_float * max(1, len(self.groups)))()
        check(_lib.mgw_pipeline_group_times(self.handle, out))
        return list(out)[: len(self.groups)]

    def close(self) -> None:
        for h in getattr(self, "_hooks", []):
            h.remove()
        self._hooks = []
        if self.ce is not None:
            self.ce.close()
            self.ce = None
        if self.handle:
            check(_lib.mgw_pipeline_destroy(self.handle))
            self.handle = None
        self.dplan.close()


def autotune_plan(model: torch.nn.Module, comm: Comm, lr: float, trace, step: Callable[[], None],
                  params: Optional[List[torch.nn.Parameter]] = None, scales=(1, 3, 10, 30, 100, 300),
                  iters: int = 8, warmup: int = 3, **kw):
    """In-situ calibration of the merge plan for a real training loop.

    The planner's cost model is the reference's `a + b*M` (comm_model.hpp:
    194-199); its `(a, b)` come from an isolated copy-engine sweep
    (`Comm.calibrate_ce`). In a host-bound training loop a group also costs
    host time on the critical path, which that sweep cannot see, so the
    effective `a` is larger. This runs the loop for `iters` steps under the
    reference `optimal_plan` (planner.hpp:63-98) with `a` scaled by each of
    `scales` (distinct plans only), times each on the device (max over
    ranks, so every rank picks the same plan) and returns
    (best plan, {scale: (groups, ms)}). `step()` must run one iteration with
    the MGWFBP object passed to it via `autotune_plan.current` (begin, forward,
    backward, end). The steps train the model (SGD is applied)."""
    import statistics

    import torch.distributed as dist

    from .gradsched import AllReduceModel, CommMeasurement, fit_model, optimal_plan

    params = list(params) if params is not None else [p for p in model.parameters() if p.requires_grad]
    counts = [p.numel() for p in params]
    sizes = [4096 << k for k in range(0, 20, 2) if (4096 << k) <= 4 * padded_elems(counts)]
    meas = comm.calibrate_ce(sizes, warmup=2, reps=5)
    t = torch.tensor([m.time_sec for m in meas], dtype=torch.float64, device=params[0].device)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    base = fit_model([CommMeasurement(m.size_bytes, float(v)) for m, v in zip(meas, t.tolist())])
    results, seen, best = {}, set(), None
    for sc in scales:
        plan = optimal_plan(trace, AllReduceModel(base.a * sc, base.b))
        key = tuple(int(x) for x in plan.tags)
        if key in seen:
            continue
        seen.add(key)
        sync = MGWFBP(model, comm, lr, plan=plan, params=params, **kw)
        autotune_plan.current = sync
        for _ in range(warmup):
            step()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
        evs[0].record()
        for i in range(iters):
            step()
            evs[i + 1].record()
        torch.cuda.synchronize()
        ms = torch.tensor([statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(iters))],
                          dtype=torch.float64, device=params[0].device)
        if dist.is_initialized():
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        sync.check()
        sync.close()
        results[sc] = (len(plan.groups()), float(ms.item()))
        if best is None or results[sc][1] < best[1]:
            best = (plan, results[sc][1])
    autotune_plan.current = None
    return best[0], results
