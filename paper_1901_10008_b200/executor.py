"""Coalesced B200 executor: one persistent sm_100a launch per scheduler step.

The reference turns each dispatch into a simulated completion at
`d.end` (gpumux/engine.py:359-364). Here a step's dispatches really run:

    ex = Executor()                                # device = current CUDA device
    ops = ex.operands_for(kernel)                  # or bring your own tensors
    ex.bind(kernel.kernel_id, ex.register_gemm(a, bt, c, bias=..., activation="relu"))
    ...
    dispatches, withheld, wakeup = scheduler.step(now)
    ex.launch_dispatches(dispatches)               # ONE kernel for all members of all dispatches

Members run at their true dims (padding is only billed by the decision model).
The work is done by libgmx_exec.so (include/gmx_exec.h); this module only
validates torch tensors and marshals pointers. There is no CPU or eager
fallback: without an sm_100 GPU or the library, construction raises.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _build, _lib

ST = {torch.bfloat16: 0, torch.float32: 1}
ACT = {"none": 0, "relu": 1, "gelu": 2}


class ProblemDesc(C.Structure):
    _fields_ = [("op", C.c_int32), ("in_dtype", C.c_int32), ("out_dtype", C.c_int32),
                ("activation", C.c_int32), ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
                ("a", C.c_void_p), ("lda", C.c_int64), ("b", C.c_void_p), ("ldb", C.c_int64),
                ("c", C.c_void_p), ("ldc", C.c_int64), ("bias", C.c_void_p),
                ("tile_n", C.c_int32), ("_reserved", C.c_int32)]


class PlanStats(C.Structure):
    _fields_ = [("grid", C.c_int32), ("n_items", C.c_int32), ("n_gemm_tiles", C.c_int32),
                ("n_split_items", C.c_int32), ("n_gemv_items", C.c_int32),
                ("n_eltwise_items", C.c_int32), ("cached", C.c_int32), ("_pad", C.c_int32),
                ("operand_bytes", C.c_int64), ("tile_load_bytes", C.c_int64),
                ("flops", C.c_int64), ("max_cta_cost", C.c_double), ("mean_cta_cost", C.c_double)]


EXEC_SIGNATURES = {
    "gmx_exec_last_error": (C.c_char_p, []),
    "gmx_exec_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "gmx_exec_destroy": (None, [C.c_void_p]),
    "gmx_exec_num_sms": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "gmx_exec_register": (C.c_int, [C.c_void_p, C.POINTER(ProblemDesc), C.POINTER(C.c_int32)]),
    "gmx_exec_unregister": (C.c_int, [C.c_void_p, C.c_int32]),
    "gmx_exec_launch": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_void_p]),
    "gmx_exec_launch_ex": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_void_p, C.c_int32]),
    "gmx_exec_last_plan": (C.c_int, [C.c_void_p, C.POINTER(PlanStats)]),
    "gmx_exec_clear_plans": (C.c_int, [C.c_void_p]),
    "gmx_exec_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "gmx_exec_resident_begin": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmx_exec_launch_deps": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                                       C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int64)]),
    "gmx_exec_resident_active": (C.c_int, [C.c_void_p]),
    "gmx_exec_resident_step_done": (C.c_int, [C.c_void_p, C.c_int64]),
    "gmx_exec_resident_end": (C.c_int, [C.c_void_p]),
    "gmx_exec_resident_begin_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "gmx_exec_resident_release": (C.c_int, [C.c_void_p]),
    "gmx_exec_resident_relay_ns": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "gmx_exec_resident_read_rtrace": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int32)]),
    "gmx_exec_resident_device_ns": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "gmx_exec_resident_completed": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "gmx_exec_resident_sm_clock": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "gmx_exec_read_trace": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32)]),
}

_exec_lib = None


def exec_lib(path=None):
    """The in-tree libgmx_exec.so. `path` (diagnostic tools only, before the first use) loads an
    instrumented build of the same ABI instead."""
    global _exec_lib
    if _exec_lib is None:
        lib = C.CDLL(path or _build.build_exec())
        for name, (res, args) in EXEC_SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _exec_lib = lib
    return _exec_lib


def _check(rc):
    if rc != 0:
        msg = (exec_lib().gmx_exec_last_error() or b"").decode(errors="replace")
        if rc == _lib.EINVAL:
            raise ValueError(msg)
        raise _lib.GmxError(f"executor error {rc}: {msg}")


def padded_ld(k: int, dtype=torch.bfloat16) -> int:
    """Leading dimension (elements) with 16-byte row strides, as TMA requires."""
    per = 16 // torch.tensor([], dtype=dtype).element_size()
    return (k + per - 1) // per * per


class Executor:
    """Registered member operands + the coalesced launch (libgmx_exec.so)."""

    def __init__(self, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("the coalesced executor needs a CUDA device (sm_100a)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self._lib = exec_lib()
        h = C.c_void_p()
        _check(self._lib.gmx_exec_create(self.device.index, C.byref(h)))
        self._h = h
        self._keep = {}            # slot -> tensors kept alive while registered
        self._kernel_slot = {}     # kernel_id -> slot
        n = C.c_int32()
        _check(self._lib.gmx_exec_num_sms(h, C.byref(n)))
        self.num_sms = n.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.gmx_exec_destroy(h)
            self._h = None

    # ---- registration ---------------------------------------------------------------

    def _check_tensor(self, t, name, dtypes):
        if t.device != self.device:
            raise ValueError(f"{name} must live on {self.device}, got {t.device}")
        if t.dtype not in dtypes:
            raise ValueError(f"{name} dtype {t.dtype} not in {dtypes}")

    def _register(self, desc, keep):
        slot = C.c_int32()
        _check(self._lib.gmx_exec_register(self._h, C.byref(desc), C.byref(slot)))
        self._keep[slot.value] = keep
        return slot.value

    def register_gemm(self, a, bt, c, bias=None, activation="none", k=None, tile_n=0):
        """C[m,n] = act(A[m,k] . Bt[n,k]^T + bias[m]); A/Bt bf16 (tcgen05 kind::f16) or fp32 (read
        as tf32, kind::tf32: the reference's "fp32" GEMMs, kernels.py:22), rows 16-byte aligned.
        tile_n: UMMA N of the output tiles (64/128; 0 = automatic, or a measured TuningTable's)."""
        self._check_tensor(a, "A", (torch.bfloat16, torch.float32))
        self._check_tensor(bt, "Bt", (a.dtype,))
        self._check_tensor(c, "C", (torch.bfloat16, torch.float32))
        m, n = c.shape
        k = a.shape[1] if k is None else k
        if a.shape[0] != m or bt.shape[0] != n or a.shape[1] < k or bt.shape[1] < k:
            raise ValueError("gemm operand shapes disagree")
        if a.stride(1) != 1 or bt.stride(1) != 1 or c.stride(1) != 1:
            raise ValueError("gemm operands must be row-major (unit inner stride)")
        d = ProblemDesc(op=_lib.OP_CODE["gemm"], in_dtype=ST[a.dtype], out_dtype=ST[c.dtype],
                        activation=ACT[activation], m=m, n=n, k=k, a=a.data_ptr(), lda=a.stride(0),
                        b=bt.data_ptr(), ldb=bt.stride(0), c=c.data_ptr(), ldc=c.stride(0),
                        bias=self._bias_ptr(bias, m), tile_n=int(tile_n))
        return self._register(d, (a, bt, c, bias))

    def register_gemv(self, w, x, y, bias=None, activation="none"):
        """y[m] = act(W[m,n] . x[n] + bias[m]); fp32 or bf16."""
        self._check_tensor(w, "W", (torch.bfloat16, torch.float32))
        self._check_tensor(x, "x", (w.dtype,))
        self._check_tensor(y, "y", (torch.bfloat16, torch.float32))
        m, n = w.shape
        if x.numel() != n or y.numel() != m or w.stride(1) != 1 or not x.is_contiguous() \
                or not y.is_contiguous():
            raise ValueError("gemv operand shapes/strides disagree")
        d = ProblemDesc(op=_lib.OP_CODE["gemv"], in_dtype=ST[w.dtype], out_dtype=ST[y.dtype],
                        activation=ACT[activation], m=m, n=n, k=1, a=w.data_ptr(), lda=w.stride(0),
                        b=x.data_ptr(), ldb=0, c=y.data_ptr(), ldc=1, bias=self._bias_ptr(bias, m))
        return self._register(d, (w, x, y, bias))

    def register_elementwise(self, x, y, activation="none"):
        """y[i] = act(x[i]) over contiguous tensors of one dtype."""
        self._check_tensor(x, "x", (torch.bfloat16, torch.float32))
        self._check_tensor(y, "y", (x.dtype,))
        if x.numel() != y.numel() or not x.is_contiguous() or not y.is_contiguous():
            raise ValueError("elementwise operands must be contiguous and equal-sized")
        d = ProblemDesc(op=_lib.OP_CODE["elementwise"], in_dtype=ST[x.dtype], out_dtype=ST[y.dtype],
                        activation=ACT[activation], m=x.numel(), n=1, k=1, a=x.data_ptr(), lda=0,
                        b=None, ldb=0, c=y.data_ptr(), ldc=0, bias=None)
        return self._register(d, (x, y))

    def _bias_ptr(self, bias, m):
        if bias is None:
            return None
        self._check_tensor(bias, "bias", (torch.float32,))
        if bias.numel() != m or not bias.is_contiguous():
            raise ValueError("bias must be a contiguous fp32 vector of length m")
        return bias.data_ptr()

    def unregister(self, slot: int):
        _check(self._lib.gmx_exec_unregister(self._h, int(slot)))
        self._keep.pop(slot, None)
        for kid in [k for k, s in self._kernel_slot.items() if s == slot]:
            del self._kernel_slot[kid]

    def bind(self, kernel_id: int, slot: int):
        """Associate a scheduler kernel id with registered operands."""
        self._kernel_slot[kernel_id] = slot

    def slot_of(self, kernel_id: int) -> int:
        return self._kernel_slot[kernel_id]

    # ---- execution ----------------------------------------------------------------------

    def launch(self, slots, stream=None, independent=False, dep_slots=None):
        """One coalesced launch over the given registered slots (async on `stream`).

        independent=True promises no member reads what the previous launch on the stream
        writes, letting this step overlap the previous step's tail (PDL). dep_slots: slots whose
        outputs the members read (their producers); in resident mode the step then waits only
        for the steps that wrote them. Returns the resident queue position (or -1)."""
        slots = list(slots)
        arr = (C.c_int32 * max(1, len(slots)))(*slots)
        deps = list(dep_slots or [])
        darr = (C.c_int32 * max(1, len(deps)))(*deps)
        seq = C.c_int64(-1)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.gmx_exec_launch_deps(self._h, arr, len(slots), darr, len(deps),
                                              C.c_void_p(s.cuda_stream), 1 if independent else 0,
                                              C.byref(seq)))
        return seq.value

    def resident_step_done(self, seq: int) -> bool:
        return bool(self._lib.gmx_exec_resident_step_done(self._h, int(seq)))

    def launch_dispatches(self, dispatches, stream=None):
        """Execute every member of every dispatch of one scheduler step in ONE launch."""
        self.launch([self._kernel_slot[kid] for d in dispatches for kid in d.kernel_ids], stream)

    def last_plan(self) -> dict:
        st = PlanStats()
        _check(self._lib.gmx_exec_last_plan(self._h, C.byref(st)))
        return {name: getattr(st, name) for name, _ in PlanStats._fields_ if name != "_pad"}

    # ---- resident (persistent) mode --------------------------------------------------

    def resident_begin(self, stream=None, hold=False):
        """Launch the persistent coalesced kernel on `stream`; until resident_end(), every
        launch() appends its step to the kernel's queue instead of launching (include/gmx_exec.h).
        hold=True: nothing runs until resident_release() (device-only timing of a queued batch)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.gmx_exec_resident_begin_ex(self._h, C.c_void_p(s.cuda_stream), 1 if hold else 0))

    def resident_release(self):
        _check(self._lib.gmx_exec_resident_release(self._h))

    def resident_device_ns(self) -> int:
        """Device time (ns, %globaltimer) from the (released) start to the last step's completion."""
        n = C.c_int64()
        _check(self._lib.gmx_exec_resident_device_ns(self._h, C.byref(n)))
        return n.value

    def resident_sm_clock(self):
        """(MHz, span ns): the SM clock over the last residency, measured on the device."""
        mhz, ns = C.c_double(), C.c_int64()
        _check(self._lib.gmx_exec_resident_sm_clock(self._h, C.byref(mhz), C.byref(ns)))
        return mhz.value, ns.value

    def _relay_ns(self) -> int:
        """Diagnostics: %globaltimer from step 0's relay to the dispatcher's latest relay (valid
        after resident_device_ns)."""
        n = C.c_int64()
        _check(self._lib.gmx_exec_resident_relay_ns(self._h, C.byref(n)))
        return n.value

    def resident_end(self):
        """Queue the stop step; work later on the resident stream is ordered after all steps."""
        _check(self._lib.gmx_exec_resident_end(self._h))

    def resident_completed(self) -> int:
        """Number of queued steps (from the start of residency) that have fully completed."""
        n = C.c_int64()
        _check(self._lib.gmx_exec_resident_completed(self._h, C.byref(n)))
        return n.value

    def resident(self, stream=None):
        """Context manager: `with ex.resident(stream): ...launches...`."""
        ex = self

        class _Ctx:
            def __enter__(self):
                ex.resident_begin(stream)
                return ex

            def __exit__(self, *exc):
                ex.resident_end()
                return False
        return _Ctx()

    def set_option(self, name: str, value: int):
        _check(self._lib.gmx_exec_set_option(self._h, name.encode(), int(value)))

    def read_trace(self):
        """Per-item %globaltimer stamps of the last launch (set_option("trace", 1) first).

        Returns (items, cta_off) with items = list of dicts: problem, type, row0, col0, kb0,
        kb1, split, nsplit, cta, t_prod, t_mma_done, t_epi, t_end (ns, absolute)."""
        n, grid = C.c_int32(), C.c_int32()
        _check(self._lib.gmx_exec_read_trace(self._h, None, None, None, 0, C.byref(n), C.byref(grid)))
        stamps = (C.c_uint64 * (8 * (max(1, n.value) + grid.value)))()
        raw = (C.c_int32 * (8 * max(1, n.value)))()
        off = (C.c_int32 * (grid.value + 1))()
        _check(self._lib.gmx_exec_read_trace(self._h, stamps, raw, off, n.value + grid.value, C.byref(n),
                                             C.byref(grid)))
        # per-CTA kernel stamps: entry, prologue done, role loops done, exit
        self.kernel_stamps = [tuple(stamps[8 * (n.value + c) + j] for j in range(4)) for c in range(grid.value)]
        cta_of = {}
        for c in range(grid.value):
            for i in range(off[c], off[c + 1]):
                cta_of[i] = c
        items = []
        for i in range(n.value):
            w = raw[8 * i: 8 * i + 8]
            packed = w[1] & 0xFFFFFFFF
            items.append({"problem": w[0], "type": packed & 0xFF, "nsplit": (packed >> 8) & 0xFF,
                          "split": (packed >> 16) & 0xFF, "row0": w[2], "col0": w[3], "kb0": w[4],
                          "kb1": w[5], "cta": cta_of.get(i, -1),
                          "t_prod": stamps[8 * i], "t_mma_done": stamps[8 * i + 1],
                          "t_epi": stamps[8 * i + 2], "t_end": stamps[8 * i + 3],
                          "t_e_start": stamps[8 * i + 4], "t_e_staged": stamps[8 * i + 5],
                          "t_e_bar": stamps[8 * i + 6], "t_e_issued": stamps[8 * i + 7]})
        return items, list(off)

    def clear_plans(self):
        _check(self._lib.gmx_exec_clear_plans(self._h))


class OperandSet:
    """Synthetic per-kernel operands in the executor's HBM layout (bench / tests).

    gemm:  A[m, lda] ~ N(0,1)/sqrt(k), Bt[n, ldb] ~ N(0,1), C[m, n]: bf16 operands for the
           reference's "fp16" kernels, fp32 operands (tf32 UMMA, fp32 C) for its "fp32" ones
    gemv:  W[m, n] ~ U(-1,1), x[n] ~ U(-1,1), y[m]   (fp32 or bf16)
    elementwise: x[n] ~ N(0,1), y[n]
    lda/ldb are padded to 16-byte rows; the pad columns hold garbage (NaN) on
    purpose so a kernel that reads past k is caught by the parity tests.
    """

    def __init__(self, op_kind, dims, dtype="fp16", device="cuda", seed=0, out_dtype=None,
                 bias=False, activation="none", on_device=False):
        if on_device:   # large synthetic workloads: generate on the GPU (no host RNG / copies)
            return self._init_on_device(op_kind, dims, dtype, device, seed, out_dtype, activation)
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.op_kind, self.dims, self.activation = op_kind, tuple(dims), activation
        st = torch.bfloat16 if dtype == "fp16" else torch.float32
        self.storage = st
        if op_kind == "gemm":
            m, n, k = dims
            ld = padded_ld(k, st)
            a = torch.full((m, ld), float("nan"), dtype=st)
            a[:, :k] = (torch.randn(m, k, generator=g) / k ** 0.5).to(st)
            bt = torch.full((n, ld), float("nan"), dtype=st)
            bt[:, :k] = torch.randn(n, k, generator=g).to(st)
            self.a, self.b = a.to(device), bt.to(device)
            odt = out_dtype or st
            # C rows padded to 16 bytes so the epilogue can TMA-store whole tiles
            self.c = torch.empty(m, padded_ld(n, odt), dtype=odt, device=device)[:, :n]
            self.bias = (torch.randn(m, generator=g) * 0.1).to(device) if bias else None
        elif op_kind == "gemv":
            m, n = dims
            self.a = (torch.rand(m, n, generator=g) * 2 - 1).to(st).to(device)
            self.b = (torch.rand(n, generator=g) * 2 - 1).to(st).to(device)
            self.c = torch.empty(m, dtype=out_dtype or st, device=device)
            self.bias = (torch.randn(m, generator=g) * 0.1).to(device) if bias else None
        else:
            (n,) = dims
            self.a = torch.randn(n, generator=g).to(st).to(device)
            self.b = None
            self.c = torch.empty(n, dtype=st, device=device)
            self.bias = None

    def _init_on_device(self, op_kind, dims, dtype, device, seed, out_dtype, activation):
        g = torch.Generator(device=device).manual_seed(seed)
        self.op_kind, self.dims, self.activation, self.bias = op_kind, tuple(dims), activation, None
        st = torch.bfloat16 if dtype == "fp16" else torch.float32
        self.storage = st
        if op_kind == "gemm":
            m, n, k = dims
            ld = padded_ld(k, st)
            self.a = (torch.randn(m, ld, generator=g, device=device) / k ** 0.5).to(st)
            self.b = torch.randn(n, ld, generator=g, device=device).to(st)
            odt = out_dtype or st
            self.c = torch.empty(m, padded_ld(n, odt), dtype=odt, device=device)[:, :n]
        elif op_kind == "gemv":
            m, n = dims
            self.a = (torch.rand(m, n, generator=g, device=device) * 2 - 1).to(st)
            self.b = (torch.rand(n, generator=g, device=device) * 2 - 1).to(st)
            self.c = torch.empty(m, dtype=out_dtype or st, device=device)
        else:
            (n,) = dims
            self.a = torch.randn(n, generator=g, device=device).to(st)
            self.b = None
            self.c = torch.empty(n, dtype=st, device=device)

    @classmethod
    def from_tensors(cls, op_kind, dims, a, b, c, bias=None, activation="none"):
        """Wrap caller-allocated operands (e.g. views into a tenant arena)."""
        self = cls.__new__(cls)
        self.op_kind, self.dims, self.activation = op_kind, tuple(dims), activation
        self.storage = a.dtype
        self.a, self.b, self.c, self.bias = a, b, c, bias
        return self

    def register(self, ex: Executor, tile_n=0) -> int:
        if self.op_kind == "gemm":
            return ex.register_gemm(self.a, self.b, self.c, self.bias, self.activation,
                                    k=self.dims[2], tile_n=tile_n)
        if self.op_kind == "gemv":
            return ex.register_gemv(self.a, self.b, self.c, self.bias, self.activation)
        return ex.register_elementwise(self.a, self.c, self.activation)

    def host_inputs(self):
        """CPU copies of the operands (for the oracle)."""
        out = {"a": self.a.cpu(), "b": None if self.b is None else self.b.cpu(),
               "bias": None if self.bias is None else self.bias.cpu()}
        return out
