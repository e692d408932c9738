"""OoO coalescing scheduler (drop-in for gpumux.scheduler).

`Scheduler` keeps the reference's public surface (scheduler.py:130-471):
the same constructor, methods, return types and the attributes the reference
tests and engine touch (`ready`, `in_flight`, `free_sms`, `predicted`,
`requests`, `params`, `_ratio_windows`). Every decision — intake prediction,
slack, clustering, withhold/stagger, SM gating, completion and dependency
unlock, eviction — is taken by the native state machine behind
`gmx_sched_*` (include/gmx_core.h). This class only marshals objects across
the C ABI and mirrors the resulting state as Python dicts; the one piece that
stays in Python is the straggler ratio window, which is off the hot path and
which the reference's tests poke directly.

All five policy variants are supported (the fifo/edf/time-mux/space-mux
baselines run in the same native core), so `compare()`-style harnesses can
swap the whole scheduler.
"""

from __future__ import annotations

import ctypes as C
import math
from collections import deque
from dataclasses import dataclass, field

from . import _lib
from .coalesce import DEFAULT_PAD_BUDGET
from .device import tuning_model_constants
from .kernels import kernel_desc
from .tuning import native_table

POLICY_VARIANTS = ("fifo", "edf", "ooo", "time-mux", "space-mux")


@dataclass(frozen=True)
class PolicyParams:
    pad_budget: float = DEFAULT_PAD_BUDGET
    max_delay_fraction: float = 0.5
    straggler_threshold: float = 2.0
    eviction_window: int = 32
    eviction_min_samples: int = 8
    jitter_width: float = 0.15
    stagger_horizon: int = 10_000  # ns a withheld cluster waits for partners
    duration_noise: float = 0.0

    def __post_init__(self):
        if not 0.0 <= self.pad_budget < 1.0:
            raise ValueError("pad_budget must be in [0, 1)")
        if not 0.0 <= self.max_delay_fraction <= 1.0:
            raise ValueError("max_delay_fraction must be in [0, 1]")
        if self.straggler_threshold <= 0:
            raise ValueError("straggler_threshold must be positive")
        if self.stagger_horizon < 1:
            raise ValueError("stagger_horizon must be >= 1 ns")


@dataclass(frozen=True)
class SchedulerPolicy:
    variant: str
    params: PolicyParams = field(default_factory=PolicyParams)

    def __post_init__(self):
        if self.variant not in POLICY_VARIANTS:
            raise ValueError(f"unknown policy {self.variant!r}; choose from {POLICY_VARIANTS}")


@dataclass(frozen=True)
class TimelineEntry:
    start: int
    end: int
    sm_allocation: int
    payload: str
    context_id: str


@dataclass
class Dispatch:
    dispatch_id: int
    kernel_ids: tuple
    super_id: str | None
    stream_ids: tuple
    start: int
    end: int
    sm_allocation: int
    context_id: str
    ctx_switch: bool
    useful_flops: int
    padded_flops: int
    predicted_duration: int
    duration: int
    infeasible: bool = False

    def timeline_entry(self) -> TimelineEntry:
        return TimelineEntry(start=self.start, end=self.end, sm_allocation=self.sm_allocation,
                             payload=self.super_id or ",".join(map(str, self.kernel_ids)),
                             context_id=self.context_id)


@dataclass
class EvictionRecord:
    stream_id: str
    time: int
    cancelled_dispatch_ids: tuple
    evicted_request_ids: tuple


@dataclass
class CompletionInfo:
    dispatch: Dispatch
    finished_requests: list  # (request, completion_time)


def slack(kernel, now: int, predicted_remaining: int) -> int:
    """Deadline minus now minus predicted remaining critical-path work."""
    if predicted_remaining < 0:
        raise ValueError("predicted_remaining must be >= 0")
    return kernel.deadline - now - predicted_remaining


@dataclass
class _RequestState:
    request: object
    remaining: set
    evicted: bool = False
    completed_at: int | None = None


class Scheduler:
    """Native OoO/coalescing state machine with the reference's Python API."""

    def __init__(self, profile, policy, tuning_table=None, jitter_rng=None):
        self.profile = profile
        self.policy = policy
        self.params = policy.params
        self.table = tuning_table
        self.jitter_rng = jitter_rng
        self._lib = _lib.core()
        p = self.params
        cparams = _lib.PolicyParamsC(float(p.pad_budget), float(p.max_delay_fraction),
                                     float(p.straggler_threshold), int(p.eviction_window),
                                     int(p.eviction_min_samples), float(p.jitter_width),
                                     int(p.stagger_horizon), float(p.duration_noise))
        model = tuning_model_constants()
        state = int(getattr(jitter_rng, "_state", 0)) if jitter_rng is not None else 0
        thandle, self._table_keep = native_table(tuning_table)
        h = C.c_void_p()
        _lib.check(self._lib.gmx_sched_create(
            C.byref(_lib.profile_struct(profile)), _lib.POLICY_CODE[policy.variant],
            C.byref(cparams), thandle, float(model["base_efficiency"]),
            float(model["footprint_slope"]), state, C.byref(h)))
        self._h = h
        self._uses_rng = policy.variant == "space-mux" or p.duration_noise > 0
        self._stream_code: dict = {}
        self._stream_name: list = []
        self._kernels: dict = {}       # kernel_id -> KernelSpec (every registered kernel)
        self._owner: dict = {}         # kernel_id -> request_id
        self.requests: dict = {}
        self.ready: dict = {}
        self.blocked: dict = {}
        self.predicted: dict = {}
        self.in_flight: dict = {}
        self.completed_kernels: set = set()
        self.evicted_streams: set = set()
        self._ratio_windows: dict = {}
        self._view = _lib.StepView()
        self._cview = _lib.CompleteView()
        self._eview = _lib.EvictView()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.gmx_sched_destroy(h)
            self._h = None

    # ---- native handle helpers --------------------------------------------

    def _code(self, stream_id) -> int:
        code = self._stream_code.get(stream_id)
        if code is None:
            out = C.c_int32()
            _lib.check(self._lib.gmx_sched_intern_stream(self._h, str(stream_id).encode(),
                                                         C.byref(out)))
            code = out.value
            self._stream_code[stream_id] = code
            self._stream_name.append(stream_id)
        return code

    def _sync_rng_out(self):
        if self._uses_rng and self.jitter_rng is not None and hasattr(self.jitter_rng, "_state"):
            st = C.c_uint64()
            self._lib.gmx_sched_jitter_state(self._h, C.byref(st))
            self.jitter_rng._state = st.value

    @property
    def free_sms(self) -> int:
        out = C.c_int64()
        _lib.check(self._lib.gmx_sched_free_sms(self._h, C.byref(out)))
        return out.value

    @free_sms.setter
    def free_sms(self, value: int):
        _lib.check(self._lib.gmx_sched_set_free_sms(self._h, int(value)))

    # ---- intake ------------------------------------------------------------

    def add_request(self, request) -> bool:
        """Register a request; False if its stream was evicted."""
        kernels = tuple(request.kernels)
        self.requests[request.request_id] = _RequestState(
            request=request, remaining={k.kernel_id for k in kernels})
        scode = self._code(request.stream_id)
        n = len(kernels)
        descs = (_lib.KernelDesc * max(n, 1))()
        offsets = (C.c_int32 * (n + 1))()
        deps = []
        for i, k in enumerate(kernels):
            descs[i] = kernel_desc(k, self._code(k.stream_id))
            deps.extend(k.deps)
            offsets[i + 1] = len(deps)
        dep_arr = (C.c_int64 * max(len(deps), 1))(*deps)
        pred = (C.c_int64 * max(n, 1))()
        accepted = C.c_int32()
        _lib.check(self._lib.gmx_sched_add_request(
            self._h, int(request.request_id), scode, int(request.arrival), descs, n, dep_arr,
            offsets, pred, C.byref(accepted)))
        if not accepted.value:
            self.requests[request.request_id].evicted = True
            return False
        for i, k in enumerate(kernels):
            kid = k.kernel_id
            self._kernels[kid] = k
            self._owner[kid] = request.request_id
            self.predicted[kid] = pred[i]
            if k.deps:
                self.blocked[kid] = k
            else:
                self.ready[kid] = k
        return True

    def predicted_remaining(self, kernel) -> int:
        out = C.c_int64()
        _lib.check(self._lib.gmx_sched_predicted_remaining(self._h, int(kernel.kernel_id),
                                                           C.byref(out)))
        return out.value

    def kernel_slack(self, kernel, now: int) -> int:
        out = C.c_int64()
        _lib.check(self._lib.gmx_sched_kernel_slack(self._h, int(kernel.kernel_id), int(now),
                                                    C.byref(out)))
        return out.value

    # ---- dispatch ------------------------------------------------------------

    def _dispatch_obj(self, rec, kids) -> Dispatch:
        streams = tuple(sorted({self._kernels[k].stream_id for k in kids}))
        ctx = "jit" if rec.context == _lib.CONTEXT_JIT else self._stream_name[rec.context]
        return Dispatch(dispatch_id=rec.dispatch_id, kernel_ids=kids,
                        super_id=("sk-" + "-".join(map(str, kids))) if rec.is_super else None,
                        stream_ids=streams, start=rec.start, end=rec.end,
                        sm_allocation=rec.sm_allocation, context_id=ctx,
                        ctx_switch=bool(rec.ctx_switch), useful_flops=rec.useful_flops,
                        padded_flops=rec.padded_flops,
                        predicted_duration=rec.predicted_duration, duration=rec.duration,
                        infeasible=bool(rec.infeasible))

    def step(self, now: int):
        """Advance the policy; returns (dispatches, withheld, wakeup_time)."""
        v = self._view
        _lib.check(self._lib.gmx_sched_step(self._h, int(now), C.byref(v)))
        dispatches = []
        if v.n_dispatches:
            kid_ptr = v.dispatch_kernel_ids
            for i in range(v.n_dispatches):
                rec = v.dispatches[i]
                kids = tuple(kid_ptr[rec.kernel_offset:rec.kernel_offset + rec.n_kernels])
                d = self._dispatch_obj(rec, kids)
                for kid in kids:
                    self.ready.pop(kid, None)
                self.in_flight[d.dispatch_id] = d
                dispatches.append(d)
        withheld = []
        if v.n_withheld:
            off, ids = v.withheld_offsets, v.withheld_kernel_ids
            withheld = [tuple(ids[off[i]:off[i + 1]]) for i in range(v.n_withheld)]
        if self._uses_rng:
            self._sync_rng_out()
        return dispatches, withheld, (v.wakeup if v.has_wakeup else None)

    # ---- completion / eviction ---------------------------------------------------

    def complete(self, dispatch_id: int, now: int) -> CompletionInfo:
        cv = self._cview
        rc = self._lib.gmx_sched_complete(self._h, int(dispatch_id), int(now), C.byref(cv))
        if rc == _lib.ENOTFOUND:
            raise KeyError(dispatch_id)
        _lib.check(rc)
        dispatch = self.in_flight.pop(dispatch_id)
        finished = []
        for i in range(cv.n_finished):
            st = self.requests[cv.finished_request_ids[i]]
            st.completed_at = now
            finished.append((st.request, now))
        for kid in dispatch.kernel_ids:
            self.completed_kernels.add(kid)
            st = self.requests.get(self._owner.get(kid))
            if st is not None:
                st.remaining.discard(kid)
        for i in range(cv.n_unlocked):
            kid = cv.unlocked_kernel_ids[i]
            self.ready[kid] = self.blocked.pop(kid, None) or self._kernels[kid]
        ratio = dispatch.duration / max(dispatch.predicted_duration, 1)
        for stream in dispatch.stream_ids:
            self._ratio_windows.setdefault(
                stream, deque(maxlen=self.params.eviction_window)).append(ratio)
        return CompletionInfo(dispatch=dispatch, finished_requests=finished)

    def straggler_ratio(self, stream_id: str):
        """p99 (nearest rank) of observed/predicted duration over the window."""
        window = self._ratio_windows.get(stream_id)
        if not window or len(window) < self.params.eviction_min_samples:
            return None
        ordered = sorted(window)
        return ordered[max(1, math.ceil(0.99 * len(ordered))) - 1]

    def find_stragglers(self) -> list:
        out = []
        for stream in sorted(self._ratio_windows):
            if stream in self.evicted_streams:
                continue
            ratio = self.straggler_ratio(stream)
            if ratio is not None and ratio > self.params.straggler_threshold:
                out.append(stream)
        return out

    def evict_straggler(self, stream_id: str, now: int) -> EvictionRecord:
        """Cancel a degraded stream's exclusive in-flight work and drop its queues."""
        ev = self._eview
        _lib.check(self._lib.gmx_sched_evict_stream(self._h, self._code(stream_id), int(now),
                                                    C.byref(ev)))
        self.evicted_streams.add(stream_id)
        cancelled = tuple(ev.cancelled_dispatch_ids[i] for i in range(ev.n_cancelled))
        for did in cancelled:
            self.in_flight.pop(did, None)
        evicted = tuple(ev.evicted_request_ids[i] for i in range(ev.n_evicted))
        for rid in evicted:
            self.requests[rid].evicted = True
        for i in range(ev.n_dropped):
            kid = ev.dropped_kernel_ids[i]
            self.ready.pop(kid, None)
            self.blocked.pop(kid, None)
        return EvictionRecord(stream_id=stream_id, time=now, cancelled_dispatch_ids=cancelled,
                              evicted_request_ids=evicted)
