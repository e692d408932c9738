#!/usr/bin/env python
"""bench.py — coalesced execution of 16 heterogeneous batch-1 tenant streams on B200.

Workload (BASELINE.json configs[1], the metric's config):
  16 tenant streams, stream i submits one request = resnet50_like[i % 13]
  (ResNet-50 conv layers as im2col GEMMs, models.json:24-38), bf16 operands
  (decision dtype "fp16"), SLO 10 ms, all arriving together each round.

One STEP = one scheduling round of those 16 requests through the product:
native OoO decisions (gpumux scheduler.py:414-454, bit-exact, b200 decision
profile) in the native event loop (engine.py:320-367), each scheduler step's
dispatches executed as ONE persistent sm_100a launch. Virtual (lockstep)
clock: the 10 us withhold stagger is a latency policy and is not charged to
throughput. Inputs rotate over R operand replicas (R x 31 MB > 126 MB L2), so
every launch reads cold operands from HBM.

  value  useful TFLOP/s (padding excluded, engine.py:425), inputs resident in HBM
  e2e    same metric through the public API with HOST buffers: per round the
         16 activation matrices go H2D from pinned memory and the 16 outputs
         come back D2H inside the timed region.
  --impl reference   the reference's CPU path (oracle port: restated gpumux
         decisions + fp32 numpy numerics on all host cores), same config.

Multi-GPU (torchrun): tenants are independent, so every rank runs its own
16-tenant shard (weak scaling, no collective on the hot path); timing is the
max over ranks; NCCL only gathers the per-rank numbers.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "coalesced ops/sec & TFLOP/s at SLO vs sequential/stream multiplexing, 1/2/4/8 B200"
RESNET50_LIKE = [(64, 3136, 147), (64, 3136, 64), (64, 3136, 576), (256, 3136, 64), (128, 784, 256),
                 (128, 784, 1152), (512, 784, 128), (256, 196, 512), (256, 196, 2304),
                 (1024, 196, 256), (512, 49, 1024), (512, 49, 4608), (2048, 49, 512)]
N_TENANTS = 16              # tenants per GPU at N=1 (C2); N GPUs partition 16*N tenants by default
SLO_NS = 10_000_000
ROUND_NS = 1_000_000        # virtual spacing of rounds (every round completes well inside it)


def c2_shapes():
    return [RESNET50_LIKE[i % 13] for i in range(N_TENANTS)]


def tenant_set(total):
    """The box's tenant set: stream i = one batch-1 request of resnet50_like[i % 13] per round
    (C2 at 16 tenants, C5 at 512). Names sort in stream order."""
    width = max(2, len(str(total - 1)))
    return [(f"t{i:0{width}d}", RESNET50_LIKE[i % 13]) for i in range(total)]


def my_tenants(total, rank, world):
    """This rank's shard: sorted stream ids dealt round-robin (sharding.shard_streams);
    each GPU runs its own scheduler + executor over it, no collective on the hot path."""
    from paper_1901_10008_b200.sharding import shard_streams
    shape_of = dict(tenant_set(total))
    return [(sid, shape_of[sid]) for sid in shard_streams(list(shape_of), world)[rank]]


def useful_flops(shapes):
    return sum(2 * m * n * k for m, n, k in shapes)


def algorithmic_bytes(shapes, elt=2):
    return sum(elt * (m * k + k * n + m * n) for m, n, k in shapes)


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            raw = json.load(fh)
        return {"hbm_gbs": raw["hbm_gbs"], "bf16_tflops": raw["bf16_tflops"], "source": "measured"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


# ---------------------------------------------------------------- distributed plumbing

def dist_setup(gloo=False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if gloo:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def all_reduce(value, op):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([float(value)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=op)
    return t.item()


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ---------------------------------------------------------------- clocks (NVML, during the timed region)

def spin_host(ms):
    """Busy-wait on the serving core right before the window: a core that idled through the
    synchronize/barrier is clocked down (a server's loop core never is); measured ~4 us per round
    slower over a 20-round window without it."""
    t_end = time.perf_counter() + ms * 1e-3
    while time.perf_counter() < t_end:
        pass


def smt_siblings(core):
    """Hardware threads sharing `core`'s physical core (sysfs), so helper threads keep off it."""
    try:
        with open(f"/sys/devices/system/cpu/cpu{core}/topology/thread_siblings_list") as fh:
            out = set()
            for part in fh.read().strip().split(","):
                a, _, b = part.partition("-")
                out.update(range(int(a), int(b or a) + 1))
            return out
    except (OSError, ValueError):
        return {core}


class ClockSampler:
    """SM clock + clock-event reasons sampled with NVML every `period_s` in a SEPARATE process
    (pinned off the serving core and its SMT siblings), from before the timed window until after
    it: NVML / driver calls inside the bench process measurably slowed the serving loop."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
    CHILD = (
        "import sys, time, pynvml\n"
        "pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1])); per = float(sys.argv[2])\n"
        "print('max', pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)\n"
        "while True:\n"
        "    t = time.perf_counter()\n"
        "    c = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)\n"
        "    m = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)\n"
        "    print(c, m, round((time.perf_counter() - t) * 1e3, 3), flush=True)\n"
        "    time.sleep(per)\n")

    def __init__(self, device_index, period_s=0.2, avoid_core=None, allowed=None):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.device_index, self.period = device_index, period_s
        self.avoid_core = avoid_core
        self.allowed = sorted(os.sched_getaffinity(0)) if allowed is None else allowed
        self.proc, self._lines, self._t = None, [], None

    def __enter__(self):
        import subprocess
        if os.environ.get("GMX_BENCH_CLOCKS") == "0":   # experiment: no sampling at all
            return self
        self.period = float(os.environ.get("GMX_CLOCK_PERIOD_MS", self.period * 1e3)) * 1e-3
        others = set(self.allowed)
        if self.avoid_core is not None:
            others -= {self.avoid_core} | smt_siblings(self.avoid_core)
        others = others or set(self.allowed)
        try:
            self.proc = subprocess.Popen(
                [sys.executable, "-c", self.CHILD, str(self.device_index), str(self.period)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
                preexec_fn=lambda: os.sched_setaffinity(0, others))
        except OSError:
            self.proc = None
            return self

        def reader():
            # off the serving core too: a thread inherits its creator's affinity, and the
            # serving thread is pinned by now — this reader woke on the serving core every
            # sample and preempted the loop (windows up to 40 % slower, measured)
            try:
                os.sched_setaffinity(0, others)
            except OSError:
                pass
            for line in self.proc.stdout:
                self._lines.append(line.split())
        self._t = threading.Thread(target=reader, daemon=True)
        self._t.start()
        return self

    def settle(self):
        """Wait until the sampler process delivers samples, so its start-up is not in the window;
        samples from the last one before this call on are the window's."""
        t0 = time.perf_counter()
        while self.proc is not None and len(self._lines) < 2 and time.perf_counter() - t0 < 10.0:
            if self.proc.poll() is not None:
                break
            time.sleep(0.001)
        self._mark = len(self._lines)

    def __exit__(self, *exc):
        if self.proc is None:
            return
        n0 = len(self._lines)
        t0 = time.perf_counter()
        while len(self._lines) == n0 and time.perf_counter() - t0 < 3 * self.period:
            time.sleep(0.002)   # one more sample after the window
        self.proc.kill()
        self.proc.wait()
        self._t.join(timeout=2)
        for f in self._lines:
            if f and f[0] == "max":
                self.max_mhz = int(f[1])
        body = [f for f in self._lines[getattr(self, "_mark", 0) - 1 if getattr(self, "_mark", 0) else 0:]
                if len(f) == 3 and f[0] != "max"]
        self.query_ms = [float(f[2]) for f in self._lines if len(f) == 3 and f[0] != "max"]
        for c, m, _ in body:
            self.samples.append(int(c))
            for name, bit in self.REASONS.items():
                if int(m) & bit:
                    self.reasons.add(name)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        q = getattr(self, "query_ms", [])
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "nvml_query_ms": {"median": round(statistics.median(q), 3), "max": round(max(q), 3)} if q else None}


# ---------------------------------------------------------------- our arm

class C2Bench:
    def __init__(self, replicas, profile_name="b200", tuning=None, tenants=None):
        import torch

        import paper_1901_10008_b200 as gm
        from paper_1901_10008_b200 import _lib
        from paper_1901_10008_b200.executor import Executor, OperandSet
        from paper_1901_10008_b200.runtime import Runtime

        self.torch, self.gm, self._lib = torch, gm, _lib
        self.tenants = tenants or tenant_set(N_TENANTS)
        self.shapes = [shape for _, shape in self.tenants]
        self.ex = Executor()
        self.replicas = replicas
        # HBM layout: per replica, the 16 activation matrices (Bt) are views into ONE contiguous
        # arena and so are the 16 outputs (C), so a round's inputs/outputs move with a single
        # DMA each; weights (A) are per-tenant resident tensors.
        from paper_1901_10008_b200.executor import padded_ld
        self.b_offsets, off = [], 0
        for (m, n, k) in self.shapes:
            self.b_offsets.append(off)
            off += n * padded_ld(k)
        self.b_numel = off
        self.c_offsets, off = [], 0
        for (m, n, k) in self.shapes:
            self.c_offsets.append(off)
            off += m * padded_ld(n)
        self.c_numel = off
        self.b_arena = [torch.empty(self.b_numel, dtype=torch.bfloat16, device="cuda") for _ in range(replicas)]
        self.c_arena = [torch.empty(self.c_numel, dtype=torch.bfloat16, device="cuda") for _ in range(replicas)]
        self.ops = []
        for r in range(replicas):
            row = []
            for i, (m, n, k) in enumerate(self.shapes):
                src = OperandSet("gemm", (m, n, k), seed=1000 * r + i)
                ldk, ldn = padded_ld(k), padded_ld(n)
                bt = self.b_arena[r][self.b_offsets[i]:self.b_offsets[i] + n * ldk].view(n, ldk)
                bt.copy_(src.b)
                c = self.c_arena[r][self.c_offsets[i]:self.c_offsets[i] + m * ldn].view(m, ldn)[:, :n]
                row.append(OperandSet.from_tensors("gemm", (m, n, k), src.a, bt, c))
            self.ops.append(row)
        # optional measured TuningTable (tools/autotune.py): decisions use it and each member's
        # executor tile is the one measured best at its co-tenancy in the round
        self.table = None
        tiles = [0] * len(self.shapes)
        if tuning:
            from paper_1901_10008_b200.autotune import tile_n_for
            from paper_1901_10008_b200.tuning import ClusterKey, TuningTable
            self.table = TuningTable.load(tuning)
            for i, dims in enumerate(self.shapes):
                tiles[i] = tile_n_for(self.table, ClusterKey("gemm", "fp16", dims), self.shapes.count(dims))
        self.slots = [[o.register(self.ex, tile_n=tiles[i]) for i, o in enumerate(row)] for row in self.ops]
        self.profile = gm.load_profile(profile_name)
        self.policy = gm.SchedulerPolicy("ooo")
        self.rt = Runtime(self.ex, self.profile, self.policy, tuning_table=self.table)
        self.codes = [self.rt.stream_code(sid) for sid, _ in self.tenants]
        self.next_round = 0
        self.stream = torch.cuda.current_stream()

    def queue_round(self, r):
        """Submit round r's 16 requests (client side: builds the request records)."""
        _lib = self._lib
        import ctypes as C
        t0 = r * ROUND_NS
        rep = r % self.replicas
        T = len(self.shapes)
        for i, (m, n, k) in enumerate(self.shapes):
            d = (_lib.KernelDesc * 1)()
            d[0].kernel_id = r * T + i
            d[0].stream = self.codes[i]
            d[0].op = _lib.OP_CODE["gemm"]
            d[0].dtype = _lib.DT_CODE["fp16"]
            d[0].ndims = 3
            d[0].dims[0], d[0].dims[1], d[0].dims[2] = m, n, k
            d[0].arrival = t0
            d[0].deadline = t0 + SLO_NS
            off = (C.c_int32 * 2)(0, 0)
            deps = (C.c_int64 * 1)()
            sl = (C.c_int32 * 1)(self.slots[rep][i])
            self.rt.submit_raw(r * T + i, self.codes[i], t0, t0 + SLO_NS, d, 1, deps, off, sl)

    def run_rounds(self, first, count):
        return self.rt.run(until=(first + count) * ROUND_NS - 1, stream=self.stream)

    def check_round_outputs(self):
        """Parity spot-check of the last round's outputs against the oracle (smoke only)."""
        from oracle import numerics as on
        torch = self.torch
        torch.cuda.synchronize()
        bad = []
        for o in self.ops[(self.next_round - 1) % self.replicas]:
            got = o.c.float().cpu().numpy()
            ref = on.gemm(o.a.float().cpu().numpy(), o.b.float().cpu().numpy(), o.dims[2])
            if not on.within(got, ref, True):
                bad.append(o.dims)
        return bad


def time_launch_only(bench, launches):
    """Average device duration of the coalesced kernel: `launches` back-to-back launches
    (rotating operand replicas, as in the timed region) captured in a CUDA graph and replayed
    between CUDA events on the launching stream, so no host gap is counted."""
    torch = bench.torch
    s = torch.cuda.Stream()
    n = max(bench.replicas, (launches // bench.replicas) * bench.replicas)
    with torch.cuda.stream(s):
        for j in range(bench.replicas):
            bench.ex.launch(bench.slots[j], s, independent=True)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for j in range(n):
                bench.ex.launch(bench.slots[j % bench.replicas], s, independent=True)
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        s.synchronize()
    plan = bench.ex.last_plan()
    return e0.elapsed_time(e1) * 1e-3 / (reps * n), plan


def time_resident(bench, steps):
    """Average device time per step of the coalesced kernel in resident mode: `steps` steps
    (rotating operand replicas) are queued to a HELD persistent launch, then released, so they
    run back to back. Timed with CUDA events: one recorded on an idle side stream right after the
    release (the held kernel occupies the launching stream), one on the launching stream after
    the stop step, i.e. release -> kernel exit; the in-kernel %globaltimer span (release -> last
    step complete) is returned beside it."""
    torch = bench.torch
    s, side = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s):
        # resident plans (their own split: DESIGN.md §4) built and uploaded before the timed batch
        bench.ex.resident_begin(s)
        for j in range(bench.replicas):
            bench.ex.launch(bench.slots[j], s, independent=True)
        bench.ex.resident_end()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bench.ex.resident_begin(s, hold=True)
        for j in range(steps):
            bench.ex.launch(bench.slots[j % bench.replicas], s, independent=True)
        bench.ex.resident_release()
        e0.record(side)
        bench.ex.resident_end()
        e1.record(s)
        s.synchronize()
        side.synchronize()
    ev_sec = e0.elapsed_time(e1) * 1e-3 / steps
    return ev_sec, bench.ex.resident_device_ns() * 1e-9 / steps, bench.ex.last_plan()


def time_comparators(bench, rounds):
    """Time-only (sequential cuBLAS launches, one stream) and space-only (one stream per
    tenant) multiplexing of the same 16 GEMMs on the same device and operands."""
    torch = bench.torch
    views = []
    for row in bench.ops:
        views.append([(o.a[:, :o.dims[2]], o.b[:, :o.dims[2]].t(), o.c) for o in row])
    streams = [torch.cuda.Stream() for _ in range(len(bench.shapes))]
    res = {}
    for mode in ("time_only", "space_only"):
        for warm in (True, False):
            n = 3 if warm else rounds
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            main = torch.cuda.current_stream()
            for r in range(n):
                row = views[r % bench.replicas]
                if mode == "time_only":
                    for a, bt, c in row:
                        torch.mm(a, bt, out=c)
                else:
                    ev = torch.cuda.Event()
                    ev.record(main)
                    for s, (a, bt, c) in zip(streams, row):
                        s.wait_event(ev)
                        with torch.cuda.stream(s):
                            torch.mm(a, bt, out=c)
                    for s in streams:
                        done = torch.cuda.Event()
                        done.record(s)
                        main.wait_event(done)
            t1.record()
            torch.cuda.synchronize()
            if not warm:
                sec = t0.elapsed_time(t1) * 1e-3 / n
                res[mode] = {"tflops": useful_flops(bench.shapes) / sec / 1e12, "ms_per_round": sec * 1e3}
    return res


def e2e_rounds(bench, first, count):
    """Public-API round trip per round: the round's 16 activation matrices go host(pinned) ->
    HBM as ONE DMA into the replica's activation arena, decisions + the coalesced launch run,
    and the 16 outputs come back HBM -> host(pinned) as ONE DMA. Copy-in, compute and copy-out
    of consecutive rounds overlap on three streams (replicas rotate, so no round overwrites
    buffers still in use)."""
    torch = bench.torch
    host_in = bench.b_arena[0].cpu().pin_memory()
    host_out = [torch.empty(bench.c_numel, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    h2d = host_in.numel() * host_in.element_size()
    d2h = host_out[0].numel() * host_out[0].element_size()
    s_in, s_cmp, s_out = torch.cuda.Stream(), bench.stream, torch.cuda.Stream()
    done = {}

    def one(r):
        rep = r % bench.replicas
        if rep in done:                      # replica buffers free again?
            s_in.wait_event(done[rep])
        with torch.cuda.stream(s_in):
            bench.b_arena[rep].copy_(host_in, non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
        s_cmp.wait_event(ev_in)
        bench.queue_round(r)
        bench.run_rounds(r, 1)
        ev_c = torch.cuda.Event()
        ev_c.record(s_cmp)
        s_out.wait_event(ev_c)
        with torch.cuda.stream(s_out):
            host_out[r % 2].copy_(bench.c_arena[rep], non_blocking=True)
            ev_o = torch.cuda.Event()
            ev_o.record(s_out)
        done[rep] = ev_o

    for r in range(first, first + 3):
        one(r)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s_in)
    for r in range(first + 3, first + 3 + count):
        one(r)
    s_in.wait_stream(s_out)
    t1.record(s_in)
    torch.cuda.synchronize()
    sec = t0.elapsed_time(t1) * 1e-3
    return sec, h2d, d2h, first + 3 + count


def replicas_for(tenants, requested):
    """Operand replicas rotated by the timed rounds: enough that the replicas' operands exceed
    4x the 126 MB L2 (every launch reads cold operands from HBM), at most `requested`."""
    per_round = algorithmic_bytes([shape for _, shape in tenants])
    return max(2, min(requested, -(-504_000_000 // per_round)))


class CpuReference:
    """The reference's CPU path on this host: restated gpumux decisions (oracle, 1 core,
    single-threaded by design) + fp32 numerics of every dispatched member (numpy BLAS on
    all host threads)."""

    def __init__(self, shapes):
        import numpy as np

        from oracle import decisions as od
        self.od, self.shapes = od, shapes
        # decisions: the reference's own gpumux Scheduler when baseline/_ref holds it (installed
        # offline from /root/reference), else the oracle's restatement of it
        self.ref = None
        ref_dir = os.path.join(REPO, "baseline", "_ref")
        if os.path.isdir(os.path.join(ref_dir, "gpumux")):
            sys.path.insert(0, ref_dir)
            try:
                import gpumux  # noqa: F401
                from gpumux import device as gd, kernels as gk, scheduler as gs
                self.ref = (gd, gk, gs)
            except Exception:  # noqa: BLE001 — fall back to the port
                self.ref = None
        rng = np.random.default_rng(0)
        self.arrays = [(rng.standard_normal((m, k), dtype=np.float32) / math.sqrt(k),
                        rng.standard_normal((n, k), dtype=np.float32)) for m, n, k in shapes]
        with open(os.path.join(REPO, "paper_1901_10008_b200", "data", "profiles.json")) as fh:
            raw = json.load(fh)["profiles"]["b200"]
        self.prof = od.Prof(**raw)

    @property
    def decisions(self):
        return "gpumux 0.1.0 (baseline/_ref)" if self.ref else "oracle port of gpumux"

    def one_round(self):
        if self.ref:
            return self._one_round_reference()
        od, shapes, arrays = self.od, self.shapes, self.arrays
        sched = od.OracleScheduler(self.prof, "ooo")
        reqs = []
        for i, (m, n, k) in enumerate(shapes):
            kern = od.K(i, f"t{i:02d}", "gemm", (m, n, k), "fp16", frozenset(), 0, SLO_NS)
            reqs.append(od.Req(i, kern.stream_id, (kern,), 0))
            sched.add_request(reqs[-1])
        now, pending = 0, set(range(len(shapes)))
        while pending:
            launched, _held, wake = sched.step(now)
            for d in launched:
                for kid in d.kernel_ids:
                    a, bt = arrays[kid]
                    _ = a @ bt.T
                sched.complete(d.dispatch_id, d.end)
                pending -= set(d.kernel_ids)
            if not launched:
                now = wake if wake is not None else now + 1
            else:
                now = max(d.end for d in launched)


    def _one_round_reference(self):
        gd, gk, gs = self.ref
        prof = gd.DeviceProfile(**self.prof._asdict())
        sched = gs.Scheduler(prof, gs.SchedulerPolicy("ooo"))
        slo = gk.LatencyConstraint(SLO_NS)
        for i, (m, n, k) in enumerate(self.shapes):
            kern = gk.KernelSpec(i, f"t{i:02d}", "gemm", (m, n, k), "fp16", arrival=0, deadline=SLO_NS)
            sched.add_request(gk.InferenceRequest(i, kern.stream_id, (kern,), 0, slo))
        now, pending = 0, set(range(len(self.shapes)))
        while pending:
            launched, _held, wake = sched.step(now)
            for d in launched:
                for kid in d.kernel_ids:
                    a, bt = self.arrays[kid]
                    _ = a @ bt.T
                sched.complete(d.dispatch_id, d.end)
                pending -= set(d.kernel_ids)
            if not launched:
                now = wake if wake is not None else now + 1
            else:
                now = max(d.end for d in launched)


def cpu_reference_rounds(seconds_budget, shapes, threads):
    """Bounded sample of CpuReference rounds: returns (useful TFLOP/s, rounds, seconds)."""
    ref = CpuReference(shapes)
    ref.one_round()     # warm BLAS
    flops = useful_flops(shapes)
    rounds, t0 = 0, time.perf_counter()
    while True:
        ref.one_round()
        rounds += 1
        el = time.perf_counter() - t0
        if el >= seconds_budget:
            return flops * rounds / el / 1e12, rounds, el


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((p.get("num_threads", 1) for p in threadpool_info()), default=os.cpu_count())
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def read_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the coalesced kernel, from the
    newest committed `ncu --set full` summary of this workload (profiles/r*_c2_full.json)."""
    import glob
    paths = sorted(glob.glob(os.path.join(REPO, "profiles", "r*_c2_full.json")))
    if not paths:
        return None
    try:
        with open(paths[-1]) as fh:
            raw = json.load(fh)
        return raw.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def idlest_core(pool, window_s=0.2):
    """The core of `pool` with the least busy time over a short window (/proc/stat): a core that
    another process (or a busy hypervisor thread) keeps busy halves the serving loop's rate."""
    def busy():
        out = {}
        try:
            with open("/proc/stat") as fh:
                for line in fh:
                    if line.startswith("cpu") and line[3:4].isdigit():
                        f = line.split()
                        vals = [int(x) for x in f[1:]]
                        out[int(f[0][3:])] = sum(vals) - vals[3] - (vals[4] if len(vals) > 4 else 0)
        except OSError:
            pass
        return out
    a = busy()
    time.sleep(window_s)
    b = busy()
    if not a or not b:
        return pool[len(pool) // 2]
    return min(pool, key=lambda c: (b.get(c, 0) - a.get(c, 0), c))


def rank_core_pool(pool, local_rank, local_world):
    """The cores of `pool` this node-local rank may pin its serving loop to: every
    local_world-th one, so the ranks of one node never share a serving core."""
    if local_world <= 1:
        return list(pool)
    return [c for i, c in enumerate(pool) if i % local_world == local_rank % local_world] or list(pool)


def pin_serving_thread(device_index):
    """Pin the calling (serving-loop) thread to one core: the native runtime is a single-threaded
    event loop, and migrations / a shared core add run-to-run noise. The core is taken from the
    GPU's NUMA-local set (NVML CPU affinity) when known, avoiding core 0 (interrupt/housekeeping
    work lands there). Returns (previous affinity, chosen core)."""
    cpus = sorted(os.sched_getaffinity(0))
    if not cpus:
        return cpus, None
    local = []
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (max(cpus) // 64) + 1)
        local = [c for c in cpus if (words[c // 64] >> (c % 64)) & 1]
    except Exception:  # noqa: BLE001 — fall back to the allowed set
        local = []
    pool = [c for c in (local or cpus) if c != 0] or cpus
    # one serving loop per rank: ranks of one node take disjoint cores (every L-th core of the
    # NUMA-local pool), or every rank's idlest-core pick lands on the same core
    pool = rank_core_pool(pool, int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    core = idlest_core(pool)
    forced = os.environ.get("GMX_HOST_CORE")   # experiments: a fixed core, or -1 = no pinning
    if forced is not None:
        if int(forced) < 0:
            return cpus, None
        core = int(forced)
    os.sched_setaffinity(0, {core})
    # every other thread of the process (CUDA driver / torch helpers started earlier) off that core
    me = threading.get_native_id()
    rest = set(cpus) - {core} - smt_siblings(core) or set(cpus) - {core}
    try:
        for tid in os.listdir("/proc/self/task"):
            if int(tid) != me and rest:
                try:
                    os.sched_setaffinity(int(tid), rest)
                except OSError:
                    pass
    except OSError:
        pass
    return cpus, core


def run_ours(args, world, rank):
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    total_tenants = args.tenants or N_TENANTS * world
    tenants = my_tenants(total_tenants, rank, world)
    bench = C2Bench(replicas_for(tenants, args.replicas), tuning=args.tuning, tenants=tenants)
    for kv in args.exec_opt:
        k, v = kv.split("=")
        bench.ex.set_option(k, int(v))
    shapes = bench.shapes
    flops_round = useful_flops(shapes)
    args.replicas = bench.replicas
    # the serving loop's core is chosen and pinned BEFORE the warmup, so the timed rounds run on
    # a core whose caches already hold the decision core's tables (a migration right before a
    # short window cost ~5 us per round over its first rounds)
    all_cpus, host_core = pin_serving_thread(torch.cuda.current_device())
    # NVML clock/reason sampling (a separate process, recipe period 200 ms) from here until after
    # the window: an NVML client attached only around the window slowed the first launches
    clocks = ClockSampler(torch.cuda.current_device(), avoid_core=host_core, allowed=all_cpus).__enter__()
    side = torch.cuda.Stream()

    def window(first, count, timed=False):
        """K rounds through the serving loop, exactly as timed: the rounds' request records are
        queued first (client side), barrier + synchronize, then the persistent kernel is launched
        and ev0 goes on an idle side stream once the launch CALL has returned (the host API cost,
        ~15-150 us on these VMs, is server set-up; the kernel's device start-up and every step
        are inside the window), the native loop runs the rounds, the stop step is queued, ev1
        follows the kernel's exit, barrier + synchronize. Per-step launches: ev0/ev1 around."""
        for r in range(first, first + count):
            bench.queue_round(r)
        before = bench.rt.run(until=first * ROUND_NS - 1, stream=bench.stream)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if timed:
            clocks.settle()   # the sampler process has run since before the warmup
            spin_host(args.host_spin_ms)
        h0 = time.perf_counter()
        if args.launch_per_step:
            e0.record(bench.stream)
            h1 = h0
            st = bench.run_rounds(first, count)
            h2 = time.perf_counter()
        else:
            bench.ex.resident_begin(bench.stream)
            e0.record(side)
            h1 = time.perf_counter()
            st = bench.run_rounds(first, count)
            h2 = time.perf_counter()
            bench.ex.resident_end()
        e1.record(bench.stream)
        h3 = time.perf_counter()
        torch.cuda.synchronize()
        side.synchronize()
        if timed:
            clocks.__exit__(None, None, None)
        barrier()
        host = {"serving_loop_per_round": round((h2 - h1) * 1e6 / count, 3)}
        if not args.launch_per_step:
            host = {"resident_begin": round((h1 - h0) * 1e6, 1), **host, "resident_end": round((h3 - h2) * 1e6, 1)}
        return e0.elapsed_time(e1) * 1e-3, before, st, host

    # warmup: W rounds (plans cached, TMA descriptors hot, clocks up), half per-step launches,
    # half through a first residency (queue, pinned ring, upload stream allocated)
    half = args.warmup // 2
    for r in range(args.warmup):
        bench.queue_round(r)
    bench.run_rounds(0, half)
    torch.cuda.synchronize()
    if not args.launch_per_step:
        bench.ex.resident_begin(bench.stream)
    bench.run_rounds(half, args.warmup - half)
    if not args.launch_per_step:
        bench.ex.resident_end()
    torch.cuda.synchronize()
    # plan pre-population + dress rehearsal (not warmup steps, not timed): untimed copies of the
    # window, together at least one round per operand replica, so every slot set the timed
    # rounds dispatch already has its cached plan (a recurring composition's plan is built once;
    # DESIGN.md §4). Measured: the first 2-3 windows of a process run 30-50 % slower (driver-side
    # set-up of the cooperative launch, a cold serving path), later ones do not.
    first = args.warmup
    prewarm = 0
    rehearsals, rehearsal_host = [], []
    while prewarm < max(args.replicas, args.prewarm_rounds) or len(rehearsals) < 3:
        n = max(1, min(args.steps, 32))
        w = window(first, n)
        rehearsals.append(round(w[0] * 1e6 / n, 3))
        rehearsal_host.append(w[3]["serving_loop_per_round"])
        first += n
        prewarm += n
    # the timed window's first step enters an idle device and takes its slot set's latency plan
    # (executor option split_pct_idle): one more rehearsal of exactly `replicas` rounds starts on
    # the replica the timed window starts on, so that plan is cached like every other one
    if not args.launch_per_step and bench.replicas <= 64:
        w = window(first, bench.replicas)
        rehearsals.append(round(w[0] * 1e6 / bench.replicas, 3))
        rehearsal_host.append(w[3]["serving_loop_per_round"])
        first += bench.replicas
        prewarm += bench.replicas
    bench.next_round = first
    # ---- timed region: exactly K rounds -------------------------------------------------
    sec_local, before, st, host_us = window(first, args.steps, timed=True)
    dev_clock = None
    if not args.launch_per_step:   # SM clock over the window, measured on the device itself
        mhz, span = bench.ex.resident_sm_clock()
        dev_clock = {"sm_mhz": round(mhz, 1), "span_us": round(span / 1e3, 1)}
    if all_cpus:
        os.sched_setaffinity(0, set(all_cpus))
    sec = all_reduce(sec_local, torch.distributed.ReduceOp.MAX) if world > 1 else sec_local
    launches = st["launches"] - before["launches"]
    kernels = st["kernels"] - before["kernels"]
    box_flops_round = all_reduce(flops_round, torch.distributed.ReduceOp.SUM) if world > 1 else flops_round
    total_flops = box_flops_round * args.steps
    value = total_flops / sec / 1e12
    bench.next_round = first + args.steps
    bad = bench.check_round_outputs()   # parity spot-check of the timed region's last round
    nxt = first + args.steps
    # ---- dominant kernel alone -------------------------------------------------------------
    # resident: a held persistent launch runs a queued batch of steps back to back, device-timed
    # (%globaltimer, release -> last step complete); launch-per-step: CUDA graph of launches
    kern_launch_sec, _ = time_launch_only(bench, max(48, min(args.steps, 200)))
    kern_gt_sec = None
    if args.launch_per_step:
        kern_sec, plan = kern_launch_sec, bench.ex.last_plan()
    else:
        kern_sec, kern_gt_sec, plan = time_resident(bench, 1000)
    peaks = load_peaks()
    per_launch_bytes = plan["operand_bytes"]
    achieved = per_launch_bytes / kern_sec / 1e9
    # ---- end to end through the public API ---------------------------------------------------
    e2e_sec, h2d, d2h, nxt = e2e_rounds(bench, nxt, max(10, min(args.steps, 50)))
    e2e_rounds_n = max(10, min(args.steps, 50))
    e2e_val = flops_round * e2e_rounds_n / e2e_sec / 1e12
    comm = None
    if world > 1:
        import torch.distributed as dist
        e2e_sec_max = all_reduce(e2e_sec, dist.ReduceOp.MAX)
        e2e_val = box_flops_round * e2e_rounds_n / e2e_sec_max / 1e12
        # end-of-run gather of per-rank numbers (the only collective; never on the hot path)
        from paper_1901_10008_b200.sharding import gather_rank_stats
        per_rank = gather_rank_stats({"rank": rank, "tenants": len(tenants), "seconds": sec_local,
                                      "flops_per_round": flops_round, "slo_misses": st["slo_misses"],
                                      "device": torch.cuda.get_device_name()})
        comm = {"backend": dist.get_backend(), "world": world,
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                "collectives": "all_reduce(MAX time, SUM flops) + all_gather_object after the timed region",
                "ranks": per_rank}
    # ---- comparators + CPU baseline (rank 0, N=1 only) ------------------------------------------
    comps, cpu = None, None
    if rank == 0 and world == 1 and not args.quick:
        comps = time_comparators(bench, max(20, min(args.steps, 200)))
        thr = blas_threads()
        cv, cr, cs = cpu_reference_rounds(args.cpu_seconds, shapes, thr)
        cpu = {"value": cv, "unit": "TFLOP/s", "cores": thr, "kind": "port",
               "sample": f"{cr} rounds of the C2 workload in {cs:.1f}s: OoO decisions by "
                         f"{CpuReference(shapes[:1]).decisions} (python, 1 core) + fp32 numpy GEMMs of "
                         f"every dispatched member ({thr} BLAS threads; the reference has no numerics)"}
    if rank != 0:
        return
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3 / args.steps, 5),
        "higher_is_better": True,
        "scaling": "strong" if args.tenants else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic operands (A~N(0,1)/sqrt(k), B~N(0,1)), shapes of resnet50_like",
        "config": {"workload": (f"C2: {total_tenants} tenant streams x 1 batch-1 request/round"
                                if total_tenants == N_TENANTS * world else
                                f"C5: {total_tenants} tenant streams x 1 batch-1 request/round")
                               + (f", partitioned over {world} GPUs ({len(tenants)} on rank 0)" if world > 1 else "")
                               + ", resnet50_like[i%13] im2col GEMMs, bf16, SLO 10ms",
                   "tenants": total_tenants,
                   "policy": "ooo (native core, bit-exact vs gpumux)", "decision_profile": "b200",
                   "tuning_table": args.tuning or "none (reference default tiles)",
                   "window": "CUDA events: ev0 on an idle side stream right after the persistent "
                             "kernel's launch call returned (device start-up inside), ev1 after its exit; "
                             "barrier + synchronize before and after" if not args.launch_per_step else
                             "CUDA events around K rounds of per-step launches; barrier + synchronize around",
                   "step": "one scheduling round in lockstep virtual time; each scheduler step "
                           "with dispatches = one coalesced step of the resident sm_100a kernel",
                   "l2": f"inputs rotate over {args.replicas} operand replicas "
                         f"({args.replicas * algorithmic_bytes(shapes) / 1e6:.0f} MB > 126 MB L2)",
                   "parallelism": f"tenant-shard x{world} (no hot-path collective)",
                   "untimed_rehearsal_rounds": prewarm},
        "ops_per_s": round(total_tenants * args.steps / sec, 1),
        "steps_dispatched": launches,
        "launches_per_step": (launches / args.steps) if args.launch_per_step else round(1 / args.steps, 5),
        "slo_misses": st["slo_misses"],
        "gpu_launches": launches if args.launch_per_step else 1,
        "host_core": host_core,
        "host_us": host_us,
        "rehearsal_us_per_round": rehearsals,
        "rehearsal_host_loop_us_per_round": rehearsal_host,
        "executor": "launch per step" if args.launch_per_step else
                    "resident (one persistent launch; steps queued through pinned host ring)",
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                     "traffic": read_traffic(),
                     "kernel": "gmx::coalesced_step_kernel",
                     "kernel_us": round(kern_sec * 1e6, 3),
                     "kernel_us_launch_per_step": round(kern_launch_sec * 1e6, 3),
                     "kernel_us_globaltimer": None if kern_gt_sec is None else round(kern_gt_sec * 1e6, 3),
                     "timing": "resident: held batch of 1000 queued steps, CUDA events release -> kernel "
                               "exit, per step" if not args.launch_per_step
                               else "CUDA graph of launches, CUDA events",
                     "algorithmic_bytes_per_launch": per_launch_bytes,
                     "peak_source": peaks["source"] + " (MEASURED_PEAKS.json hbm_gbs)",
                     "plan": {k: plan[k] for k in ("grid", "n_items", "n_gemm_tiles", "n_split_items",
                                                   "tile_load_bytes")}},
        "e2e": {"value": round(e2e_val, 3), "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "clocks": dict(clocks.summary(), **({"device_measured": dev_clock} if dev_clock else {})),
    }
    if comm:
        out["comm"] = comm
    if comps:
        out["comparators"] = {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in comps.items()}
        out["comparators"]["coalesced_vs_time_only"] = round(value / comps["time_only"]["tflops"], 2)
        out["comparators"]["coalesced_vs_space_only"] = round(value / comps["space_only"]["tflops"], 2)
    if cpu:
        out["cpu_baseline"] = {k: (round(v, 5) if isinstance(v, float) else v) for k, v in cpu.items()}
    if bad:
        out["parity_failures"] = [list(d) for d in bad]
    print(json.dumps(out), flush=True)


def run_reference(args, world, rank):
    """Reference arm: the reference's CPU implementation of the path (oracle port) on this host."""
    if rank != 0:
        return
    thr = blas_threads()
    shapes = c2_shapes()
    ref = CpuReference(shapes)
    for _ in range(args.warmup):
        ref.one_round()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.one_round()
    el = time.perf_counter() - t0
    value = useful_flops(shapes) * args.steps / el / 1e12
    out = {"metric": METRIC, "value": round(value, 5), "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el * 1e3 / args.steps, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
           "data": "synthetic operands", "impl": "reference",
           "config": {"workload": "C2: 16 tenant streams x 1 batch-1 request/round, "
                                  "resnet50_like[i%13] im2col GEMMs", "parallelism": "host CPU"},
           "cpu_baseline": {"value": round(value, 5), "unit": "TFLOP/s", "cores": thr, "kind": "port",
                            "sample": f"{args.steps} rounds: OoO decisions by {ref.decisions} + fp32 numpy "
                                      f"GEMMs of every dispatched member (the reference has no numerics)"},
           "e2e": {"value": round(value, 5), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_dry(args, world, rank):
    """--dry-run (CPU, gloo): the multi-GPU path without a GPU. Each rank takes its tenant shard,
    runs warmup + steps rounds through the native serving loop in decisions-only mode (no
    executor), checks its shard's per-request completion times against the oracle engine run on
    the same sub-workload (each shard's trace equals the reference run() on it),
    and rank 0 prints the line with whole-box numbers (sum of work / max over ranks)."""
    import torch.distributed as dist

    import paper_1901_10008_b200 as gm
    from oracle import decisions as od
    from oracle import sim
    from paper_1901_10008_b200 import _lib
    from paper_1901_10008_b200.runtime import Runtime
    from paper_1901_10008_b200.sharding import gather_rank_stats
    import ctypes as C

    total = args.tenants or N_TENANTS * world
    tenants = my_tenants(total, rank, world)
    rounds = args.warmup + args.steps
    rt = Runtime(None, gm.load_profile("b200"), gm.SchedulerPolicy("ooo"))
    codes = [rt.stream_code(sid) for sid, _ in tenants]
    T = len(tenants)
    for r in range(rounds):
        t0 = r * ROUND_NS
        for i, (_, (m, n, k)) in enumerate(tenants):
            d = (_lib.KernelDesc * 1)()
            d[0].kernel_id, d[0].stream = r * T + i, codes[i]
            d[0].op, d[0].dtype, d[0].ndims = _lib.OP_CODE["gemm"], _lib.DT_CODE["fp16"], 3
            d[0].dims[0], d[0].dims[1], d[0].dims[2] = m, n, k
            d[0].arrival, d[0].deadline = t0, t0 + SLO_NS
            rt.submit_raw(r * T + i, codes[i], t0, t0 + SLO_NS, d, 1, (C.c_int64 * 1)(),
                          (C.c_int32 * 2)(0, 0), (C.c_int32 * 1)(0))
    h0 = time.perf_counter()
    st = rt.run()
    host_sec = time.perf_counter() - h0
    got = {(tenants[rid % T][0], (rid // T) * ROUND_NS): t for rid, t in rt.drain_completions(1 << 20)}
    # oracle engine on this shard's sub-workload (same streams, same per-round arrivals)
    library = {f"m{j}": [{"op_kind": "gemm", "dims": list(s), "dtype": "fp16"}]
               for j, s in enumerate(RESNET50_LIKE)}
    workload = {"duration_ns": rounds * ROUND_NS, "streams": [
        {"stream_id": sid, "model_name": f"m{RESNET50_LIKE.index(shape)}", "slo_ns": SLO_NS,
         "arrival": {"kind": "fixed", "schedule": [r * ROUND_NS for r in range(rounds)]}}
        for sid, shape in tenants]}
    raw = json.load(open(os.path.join(REPO, "paper_1901_10008_b200", "data", "profiles.json")))
    _tr, _m, _tl, osched = sim.simulate(workload, library, od.Prof(**raw["profiles"]["b200"]), "ooo")
    want = {(st_["request"].stream_id, st_["request"].arrival): st_["done_at"] for st_ in osched.reqs.values()}
    parity = got == want and len(got) == T * rounds
    flops = useful_flops([s for _, s in tenants]) * rounds
    stats = gather_rank_stats({"rank": rank, "tenants": [sid for sid, _ in tenants], "parity": parity,
                               "flops": flops, "host_seconds": host_sec,
                               "dispatched_steps": st["launches"]})
    if rank != 0:
        return
    t_max = max(x["host_seconds"] for x in stats)
    out = {"metric": METRIC, "dry_run": True, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "value": round(sum(x["flops"] for x in stats) / t_max / 1e12, 6),
           "unit": "useful TFLOP/s of decisions (no device; host loop only)",
           "scaling": "strong" if args.tenants else "weak", "tenants": total,
           "shard_parity": all(x["parity"] for x in stats),
           "comm": {"backend": dist.get_backend() if dist.is_initialized() else None, "world": world},
           "ranks": stats}
    print(json.dumps(out), flush=True)


def spawn_ranks(n):
    """`bench.py --gpus N` run without torchrun: launch N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 and pass rank 0's output through."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--replicas", type=int, default=16,
                    help="max operand replicas rotated by the rounds (capped at 4x L2 of operands)")
    ap.add_argument("--tenants", type=int, default=0,
                    help="total tenant streams of the box, partitioned over the GPUs (default 16 per GPU; "
                         "C5 = 512)")
    ap.add_argument("--prewarm-rounds", type=int, default=0,
                    help="plan pre-population rounds before the window (at least one per replica)")
    ap.add_argument("--host-spin-ms", type=float, default=0.0,
                    help="busy-wait on the serving core before the timed window (0 = off)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: decisions-only shards over gloo (tests the multi-rank path on CPU)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--quick", action="store_true", help="skip comparators and CPU baseline")
    ap.add_argument("--tuning", default=None,
                    help="measured TuningTable JSON (tools/autotune.py) for decisions and tiles")
    ap.add_argument("--exec-opt", action="append", default=[], metavar="K=V",
                    help="executor option (gmx_exec_set_option), repeatable; experiments only")
    ap.add_argument("--launch-per-step", action="store_true",
                    help="one kernel launch per scheduler step instead of the resident executor")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world, rank, _ = dist_setup(gloo=args.dry_run)
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using {world} ranks", file=sys.stderr)
    try:
        if args.dry_run:
            run_dry(args, world, rank)
        elif args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
