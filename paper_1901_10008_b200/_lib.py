"""ctypes bindings to the two in-tree native libraries (include/gmx_core.h,
include/gmx_exec.h).

This is the reference-side binding INTEGRATION.md shows: plain C structs and
pointers, nothing torch-specific. Libraries are (re)built in-tree on first
use when missing or stale, so a fresh checkout works without a separate build
step; a failed build raises — there is no Python fallback for any decision or
compute on the product path.
"""

from __future__ import annotations

import ctypes as C
import threading

from . import _build

# ---- codes (mirror gmx_core.h) ---------------------------------------------
OK, EINVAL, ENOTFOUND, EOVERFLOW, ESTATE, ECUDA, ENOMEM = 0, -1, -2, -3, -4, -5, -6
OP_CODE = {"elementwise": 0, "gemm": 1, "gemv": 2}
OP_NAME = {v: k for k, v in OP_CODE.items()}
DT_CODE = {"fp16": 0, "fp32": 1}
PATH_CODE = {"dense": 0, "scalar": 1}
POLICY_CODE = {"fifo": 0, "edf": 1, "ooo": 2, "time-mux": 3, "space-mux": 4}
CONTEXT_JIT = -2

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER


class Profile(C.Structure):
    _fields_ = [("sm_count", i64), ("blocks_per_sm", i64), ("peak_flops_dense", f64),
                ("peak_flops_scalar", f64), ("mem_bandwidth", f64),
                ("context_switch_cost", i64)]


class PolicyParamsC(C.Structure):
    _fields_ = [("pad_budget", f64), ("max_delay_fraction", f64), ("straggler_threshold", f64),
                ("eviction_window", i64), ("eviction_min_samples", i64), ("jitter_width", f64),
                ("stagger_horizon", i64), ("duration_noise", f64)]


class TuningConfigC(C.Structure):
    _fields_ = [("tile_m", i64), ("tile_n", i64), ("sm_footprint", f64),
                ("efficiency_factor", f64)]


class KernelDesc(C.Structure):
    _fields_ = [("kernel_id", i64), ("stream", i32), ("op", i32), ("dtype", i32),
                ("ndims", i32), ("dims", i64 * 3), ("arrival", i64), ("deadline", i64)]


class CostC(C.Structure):
    _fields_ = [("flops", i64), ("bytes", i64), ("block_count", i64), ("efficiency", f64),
                ("duration", i64)]


class DispatchRec(C.Structure):
    _fields_ = [("dispatch_id", i64), ("start", i64), ("end", i64), ("useful_flops", i64),
                ("padded_flops", i64), ("predicted_duration", i64), ("duration", i64),
                ("sm_allocation", i32), ("context", i32), ("ctx_switch", i32),
                ("infeasible", i32), ("is_super", i32), ("kernel_offset", i32),
                ("n_kernels", i32), ("_pad", i32)]


class StepView(C.Structure):
    _fields_ = [("n_dispatches", i32), ("dispatches", P(DispatchRec)),
                ("dispatch_kernel_ids", P(i64)), ("n_withheld", i32),
                ("withheld_offsets", P(i32)), ("withheld_kernel_ids", P(i64)),
                ("has_wakeup", i32), ("wakeup", i64)]


class CompleteView(C.Structure):
    _fields_ = [("dispatch", DispatchRec), ("kernel_ids", P(i64)), ("n_finished", i32),
                ("finished_request_ids", P(i64)), ("n_unlocked", i32),
                ("unlocked_kernel_ids", P(i64))]


class EvictView(C.Structure):
    _fields_ = [("n_cancelled", i32), ("cancelled_dispatch_ids", P(i64)), ("n_evicted", i32),
                ("evicted_request_ids", P(i64)), ("n_dropped", i32),
                ("dropped_kernel_ids", P(i64))]


CORE_SIGNATURES = {
    "gmx_last_error": (C.c_char_p, []),
    "gmx_core_version": (C.c_int, []),
    "gmx_flop_count": (C.c_int, [i32, P(i64), i32, P(i64)]),
    "gmx_bytes_moved": (C.c_int, [i32, P(i64), i32, i32, P(i64)]),
    "gmx_block_count": (C.c_int, [i32, P(i64), i32, i64, i64, P(i64)]),
    "gmx_occupancy_efficiency": (C.c_int, [P(Profile), i64, f64, P(f64)]),
    "gmx_roofline_duration": (C.c_int, [P(Profile), i64, i64, f64, i32, P(i64)]),
    "gmx_kernel_cost": (C.c_int, [P(Profile), P(KernelDesc), P(TuningConfigC), P(CostC)]),
    "gmx_tuning_table_create": (C.c_int, [P(C.c_void_p)]),
    "gmx_tuning_table_destroy": (None, [C.c_void_p]),
    "gmx_tuning_table_put": (C.c_int, [C.c_void_p, i32, i32, P(i64), i32, i64, P(TuningConfigC)]),
    "gmx_tuning_table_lookup": (C.c_int, [C.c_void_p, i32, i32, P(i64), i32, i64,
                                          P(TuningConfigC), P(i32)]),
    "gmx_padding_waste": (C.c_int, [i32, P(i64), i32, P(i64), i32, P(f64)]),
    "gmx_cluster_shapes": (C.c_int, [P(KernelDesc), i32, f64, P(i32), P(i32), P(i64), P(f64),
                                     P(i32)]),
    "gmx_form_superkernel": (C.c_int, [P(Profile), C.c_void_p, i32, i32, P(i64), i32, i64, i64,
                                       P(CostC)]),
    "gmx_sched_create": (C.c_int, [P(Profile), i32, P(PolicyParamsC), C.c_void_p, f64, f64, u64,
                                   P(C.c_void_p)]),
    "gmx_sched_destroy": (None, [C.c_void_p]),
    "gmx_sched_intern_stream": (C.c_int, [C.c_void_p, C.c_char_p, P(i32)]),
    "gmx_sched_add_request": (C.c_int, [C.c_void_p, i64, i32, i64, P(KernelDesc), i32, P(i64),
                                        P(i32), P(i64), P(i32)]),
    "gmx_sched_step": (C.c_int, [C.c_void_p, i64, P(StepView)]),
    "gmx_sched_complete": (C.c_int, [C.c_void_p, i64, i64, P(CompleteView)]),
    "gmx_sched_set_retire": (C.c_int, [C.c_void_p, i32]),
    "gmx_sched_evict_stream": (C.c_int, [C.c_void_p, i32, i64, P(EvictView)]),
    "gmx_sched_predicted_remaining": (C.c_int, [C.c_void_p, i64, P(i64)]),
    "gmx_sched_kernel_slack": (C.c_int, [C.c_void_p, i64, i64, P(i64)]),
    "gmx_sched_free_sms": (C.c_int, [C.c_void_p, P(i64)]),
    "gmx_sched_set_free_sms": (C.c_int, [C.c_void_p, i64]),
    "gmx_sched_num_ready": (C.c_int, [C.c_void_p, P(i64)]),
    "gmx_sched_jitter_state": (C.c_int, [C.c_void_p, P(u64)]),
    "gmx_sched_set_jitter_state": (C.c_int, [C.c_void_p, u64]),
}

_lock = threading.Lock()
_core = None


class GmxError(RuntimeError):
    pass


def core():
    """The decision-core library (built in-tree on first use)."""
    global _core
    if _core is None:
        with _lock:
            if _core is None:
                lib = C.CDLL(_build.build_core())
                for name, (res, args) in CORE_SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _core = lib
    return _core


def check(rc, lib=None):
    """Map a C status to the reference's Python exception types."""
    if rc == OK:
        return
    lib = lib or core()
    msg = (lib.gmx_last_error() or b"").decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOTFOUND:
        raise KeyError(msg)
    if rc == EOVERFLOW:
        raise OverflowError(msg)
    raise GmxError(f"gmx error {rc}: {msg}")


def dims_array(dims):
    arr = (i64 * 3)()
    for i, d in enumerate(dims):
        arr[i] = d
    return arr


def profile_struct(profile):
    """Duck-typed DeviceProfile -> gmx_profile (validated by the caller's type)."""
    return Profile(int(profile.sm_count), int(profile.blocks_per_sm),
                   float(profile.peak_flops_dense), float(profile.peak_flops_scalar),
                   float(profile.mem_bandwidth), int(profile.context_switch_cost))


def config_struct(cfg):
    return TuningConfigC(int(cfg.tile_m), int(cfg.tile_n), float(cfg.sm_footprint),
                         float(cfg.efficiency_factor))
