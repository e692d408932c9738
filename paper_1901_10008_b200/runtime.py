"""Native serving loop: OoO decisions -> one coalesced launch per step.

`Runtime` couples a native scheduler handle (gmx_sched, libgmx_core.so) with
the executor (libgmx_exec.so) through gmx_runtime (include/gmx_runtime.h),
which restates the reference's event loop (gpumux/engine.py:320-367) in C++.
Per step, Python is not involved: requests are queued with `submit`, and
`run` drains events, steps the scheduler and launches every step's
dispatches as ONE kernel on the given CUDA stream.

Lockstep mode keeps the reference's virtual clock (completions at the
decision model's d.end), so the decision sequence is bit-identical to
`gpumux.engine.run` on the same arrivals while the work really executes.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .device import tuning_model_constants
from .executor import exec_lib
from .kernels import kernel_desc
from .tuning import native_table


class ReplayRec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("t", C.c_int64), ("a", C.c_int64),
                ("off", C.c_int64)]


class RuntimeStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("now", "steps", "launches", "dispatches", "kernels",
                                         "withheld", "completed_requests", "useful_flops",
                                         "slo_misses", "evicted_requests", "cancelled_dispatches")]


RT_SIGNATURES = {
    "gmx_runtime_last_error": (C.c_char_p, []),
    "gmx_runtime_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "gmx_runtime_destroy": (None, [C.c_void_p]),
    "gmx_runtime_submit": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                                     C.POINTER(_lib.KernelDesc), C.c_int32, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "gmx_runtime_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(RuntimeStats)]),
    "gmx_runtime_drain_completions": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64),
                                                C.POINTER(C.c_int64), C.c_int32,
                                                C.POINTER(C.c_int32)]),
    "gmx_runtime_set_origin": (C.c_int, [C.c_void_p, C.c_int64]),
    "gmx_runtime_set_streams": (C.c_int, [C.c_void_p, C.c_int32]),
    "gmx_runtime_clock_ns": (C.c_int64, [C.c_void_p]),
    "gmx_runtime_host_profile": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "gmx_runtime_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "gmx_runtime_set_measured_stragglers": (C.c_int, [C.c_void_p, C.c_int32]),
    "gmx_runtime_replay_log": (C.c_int, [C.c_void_p, C.POINTER(ReplayRec), C.c_int64,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int64,
                                         C.POINTER(C.c_int64)]),
}
MODES = {"lockstep": 0, "realtime": 1}

_bound = False


def _rt_lib():
    global _bound
    lib = exec_lib()
    if not _bound:
        for name, (res, args) in RT_SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return lib


def _check(rc):
    if rc != 0:
        msg = (_rt_lib().gmx_runtime_last_error() or b"").decode(errors="replace")
        raise _lib.GmxError(f"runtime error {rc}: {msg}")


class Runtime:
    """mode="lockstep": the reference's virtual clock (decisions bit-identical to
    gpumux.engine.run); mode="realtime": wall clock, completions observed from CUDA events,
    every step logged for replay parity (`replay_log`)."""

    def __init__(self, executor, profile, policy, tuning_table=None, jitter_state=0, mode="lockstep",
                 retire=True):
        self.ex = executor
        core = _lib.core()
        p = policy.params
        cparams = _lib.PolicyParamsC(float(p.pad_budget), float(p.max_delay_fraction),
                                     float(p.straggler_threshold), int(p.eviction_window),
                                     int(p.eviction_min_samples), float(p.jitter_width),
                                     int(p.stagger_horizon), float(p.duration_noise))
        model = tuning_model_constants()
        thandle, self._table_keep = native_table(tuning_table)
        h = C.c_void_p()
        _lib.check(core.gmx_sched_create(C.byref(_lib.profile_struct(profile)),
                                         _lib.POLICY_CODE[policy.variant], C.byref(cparams),
                                         thandle, float(model["base_efficiency"]),
                                         float(model["footprint_slope"]), int(jitter_state),
                                         C.byref(h)))
        self._sched = h
        # the serving loop never queries finished requests: let the core retire them so its
        # tables stay small over long runs (decisions are unchanged)
        _lib.check(core.gmx_sched_set_retire(h, 1 if retire else 0))
        rt = C.c_void_p()
        # executor None: decisions-only engine (lockstep; nothing is launched)
        _check(_rt_lib().gmx_runtime_create(h, executor._h if executor is not None else None,
                                            MODES[mode], C.byref(rt)))
        self.mode = mode
        self._rt = rt
        self._codes = {}
        self._stats = RuntimeStats()

    def __del__(self):
        try:
            if getattr(self, "_rt", None):
                _rt_lib().gmx_runtime_destroy(self._rt)
                self._rt = None
            if getattr(self, "_sched", None):
                _lib.core().gmx_sched_destroy(self._sched)
                self._sched = None
        except TypeError:   # interpreter shutdown: module globals already torn down
            pass

    def stream_code(self, name) -> int:
        code = self._codes.get(name)
        if code is None:
            out = C.c_int32()
            _lib.check(_lib.core().gmx_sched_intern_stream(self._sched, str(name).encode(),
                                                           C.byref(out)))
            code = self._codes[name] = out.value
        return code

    def submit(self, request, slots):
        """Queue a request (duck-typed InferenceRequest) whose i-th kernel runs on slots[i]."""
        ks = tuple(request.kernels)
        n = len(ks)
        descs = (_lib.KernelDesc * max(n, 1))()
        off = (C.c_int32 * (n + 1))()
        deps = []
        for i, k in enumerate(ks):
            descs[i] = kernel_desc(k, self.stream_code(k.stream_id))
            deps.extend(k.deps)
            off[i + 1] = len(deps)
        dep_arr = (C.c_int64 * max(1, len(deps)))(*deps)
        sl = (C.c_int32 * max(1, n))(*slots)
        deadline = min(k.deadline for k in ks) if ks else 0
        self.submit_raw(request.request_id, self.stream_code(request.stream_id), request.arrival,
                        deadline, descs, n, dep_arr, off, sl)

    def submit_raw(self, rid, stream_code, arrival, deadline, descs, n, dep_arr, off, slots):
        _check(_rt_lib().gmx_runtime_submit(self._rt, int(rid), int(stream_code), int(arrival),
                                            int(deadline), descs, int(n), dep_arr, off, slots))

    def run(self, until=(1 << 62), stream=None) -> dict:
        if self.ex is None:   # decisions-only engine
            handle = None
        else:
            s = stream if stream is not None else torch.cuda.current_stream(self.ex.device)
            handle = s.cuda_stream
        _check(_rt_lib().gmx_runtime_run(self._rt, int(until), C.c_void_p(handle), C.byref(self._stats)))
        return {n: getattr(self._stats, n) for n, _ in RuntimeStats._fields_}

    def set_measured_stragglers(self, on: bool):
        """Wall-clock mode: straggler windows get observed durations."""
        _check(_rt_lib().gmx_runtime_set_measured_stragglers(self._rt, 1 if on else 0))

    def set_profiling(self, on: bool):
        """Accumulate host ns per phase (host_profile); costs ~1 us per C2 round when on."""
        _check(_rt_lib().gmx_runtime_set_profiling(self._rt, 1 if on else 0))

    def host_profile(self) -> dict:
        """Cumulative host ns in the decision core (add/step/complete) and the launch path."""
        arr = (C.c_int64 * 4)()
        _check(_rt_lib().gmx_runtime_host_profile(self._rt, arr))
        return dict(zip(("add_request", "step", "complete", "launch"), list(arr)))

    def set_streams(self, n: int):
        """Realtime mode: launch over n runtime-owned CUDA streams (small steps co-run)."""
        _check(_rt_lib().gmx_runtime_set_streams(self._rt, int(n)))

    def set_origin_now(self):
        """Realtime mode: start the runtime clock now (arrival times are relative to it)."""
        import time
        _check(_rt_lib().gmx_runtime_set_origin(self._rt, time.monotonic_ns()))

    def clock_ns(self) -> int:
        return _rt_lib().gmx_runtime_clock_ns(self._rt)

    def replay_log(self):
        """[(kind, t, a, kernel_ids)] — see include/gmx_runtime.h for the record kinds."""
        lib = _rt_lib()
        n, nk = C.c_int64(), C.c_int64()
        _check(lib.gmx_runtime_replay_log(self._rt, None, 0, C.byref(n), None, 0, C.byref(nk)))
        recs = (ReplayRec * max(1, n.value))()
        kids = (C.c_int64 * max(1, nk.value))()
        _check(lib.gmx_runtime_replay_log(self._rt, recs, n.value, C.byref(n), kids, nk.value, C.byref(nk)))
        return [(r.kind, r.t, r.a, tuple(kids[r.off:r.off + r.n]) if r.kind in (2, 3) else ())
                for r in recs[:n.value]]

    def measured_durations(self) -> dict:
        """dispatch id -> the observed duration (ns) its completion fed to the straggler windows
        (wall-clock mode with set_measured_stragglers; replay-log kind 0)."""
        lib = _rt_lib()
        n, nk = C.c_int64(), C.c_int64()
        _check(lib.gmx_runtime_replay_log(self._rt, None, 0, C.byref(n), None, 0, C.byref(nk)))
        recs = (ReplayRec * max(1, n.value))()
        kids = (C.c_int64 * max(1, nk.value))()
        _check(lib.gmx_runtime_replay_log(self._rt, recs, n.value, C.byref(n), kids, nk.value, C.byref(nk)))
        return {r.a: r.off for r in recs[:n.value] if r.kind == 0 and r.off >= 0}

    def drain_completions(self, capacity=65536):
        ids = (C.c_int64 * capacity)()
        ts = (C.c_int64 * capacity)()
        n = C.c_int32()
        _check(_rt_lib().gmx_runtime_drain_completions(self._rt, ids, ts, capacity, C.byref(n)))
        return list(zip(ids[:n.value], ts[:n.value]))
