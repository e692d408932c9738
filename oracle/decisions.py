"""Decision oracle: plain-Python restatement of the gpumux decision layer.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). The product path is the
C++ core in paper_1901_10008_b200/csrc/core; this module is the independent
checker it is compared against, and the single-core CPU arm `bench.py
--impl reference` times.

Citations are `path:line` under /root/reference/pkg/src/gpumux/. The code is
written in a functional style over duck-typed inputs: a "kernel" is any
object with kernel_id / stream_id / op_kind / dims / dtype / deps / arrival /
deadline attributes (the reference's KernelSpec, the product's KernelSpec, or
`oracle.decisions.K`), a "profile" anything with the seven DeviceProfile
attributes, a "request" anything with request_id / stream_id / kernels /
arrival.
"""

from __future__ import annotations

import math
from collections import deque, namedtuple
from types import SimpleNamespace

NO_DEADLINE = 1 << 62                       # kernels.py:25
ELEM_BYTES = {"fp32": 4, "fp16": 2}          # kernels.py:22
ARITY = {"gemm": 3, "gemv": 2, "elementwise": 1}   # kernels.py:30
DEFAULT_TILE = (64, 64, 1.0, 1.0)           # tuning.py:48-49 (tm, tn, footprint, factor)
FOOTPRINT_MODEL = (0.6, 0.4)                # presets.json tuning_model (base, slope)

K = namedtuple("K", "kernel_id stream_id op_kind dims dtype deps arrival deadline")
Req = namedtuple("Req", "request_id stream_id kernels arrival")
Prof = namedtuple("Prof", "name sm_count blocks_per_sm peak_flops_dense "
                          "peak_flops_scalar mem_bandwidth context_switch_cost")
Cost = namedtuple("Cost", "flops bytes block_count efficiency duration")


# ---- L2 kernel arithmetic (kernels.py:45-69, 202-222) ---------------------

def op_flops(op, dims):
    """kernels.py:45-54 — gemm 2mnk, gemv 2mn, elementwise n."""
    if op == "gemm":
        return 2 * dims[0] * dims[1] * dims[2]
    if op == "gemv":
        return 2 * dims[0] * dims[1]
    return dims[0]


def op_bytes(op, dims, dtype):
    """kernels.py:57-69 — every operand and the result once at dtype width."""
    w = ELEM_BYTES[dtype]
    if op == "gemm":
        m, n, k = dims
        return w * (m * k + k * n + m * n)
    if op == "gemv":
        m, n = dims
        return w * (m * n + n + m)
    return w * 2 * dims[0]


def model_blocks(op, dims, tile_m, tile_n):
    """kernels.py:202-213 — model thread blocks, tile clamped to the dims.

    The reference rounds with math.ceil over a float quotient; so do we.
    """
    if op == "gemm":
        return math.ceil(dims[0] / min(tile_m, dims[0])) * \
            math.ceil(dims[1] / min(tile_n, dims[1]))
    if op == "gemv":
        return math.ceil(dims[0] / min(tile_m, dims[0]))
    return math.ceil(dims[0] / min(tile_m * tile_n, dims[0]))


# ---- L1 device model (device.py:130-150) ----------------------------------

def occupancy(profile, blocks, factor=1.0):
    """device.py:130-137."""
    cap = profile.sm_count * profile.blocks_per_sm
    return min(1.0, blocks / cap) * factor


def roofline_ns(profile, flops, nbytes, eff, path):
    """device.py:140-150 — max(compute, memory), each ceil'd to integer ns."""
    peak = profile.peak_flops_dense if path == "dense" else profile.peak_flops_scalar
    c = math.ceil(flops / (peak * eff) * 1e9) if flops else 0
    m = math.ceil(nbytes / profile.mem_bandwidth * 1e9) if nbytes else 0
    return c if c > m else m


def path_of(dtype):
    """kernels.py:122-124 — fp16 runs on the dense (tensor) path."""
    return "dense" if dtype == "fp16" else "scalar"


def solo_cost(profile, kern, cfg=DEFAULT_TILE):
    """kernels.py:216-222 (kernel_cost)."""
    f = op_flops(kern.op_kind, kern.dims)
    b = op_bytes(kern.op_kind, kern.dims, kern.dtype)
    nb = model_blocks(kern.op_kind, kern.dims, cfg[0], cfg[1])
    e = occupancy(profile, nb, cfg[3])
    return Cost(f, b, nb, e, roofline_ns(profile, f, b, e, path_of(kern.dtype)))


# ---- L3 tuning-table lookup (tuning.py:152-160) ---------------------------

def table_config(table, op, dtype, dims, tenancy):
    """tuning.py:152-160 — `table` is {(op, dtype, dims, tenancy): cfg-tuple}.

    Tenancy above the tuned maximum for the key clamps to it; any miss falls
    back to the 64x64 default.
    """
    if not table:
        return DEFAULT_TILE
    levels = [t for (o, d, s, t) in table if (o, d, s) == (op, dtype, tuple(dims))]
    if not levels:
        return DEFAULT_TILE
    top = max(levels)
    if top == 0:
        return DEFAULT_TILE
    return table.get((op, dtype, tuple(dims), min(tenancy, top)), DEFAULT_TILE)


def table_from_reference(tuning_table):
    """Convert a reference-style TuningTable (entries {(ClusterKey, t): cfg})."""
    if tuning_table is None:
        return {}
    out = {}
    for (key, t), c in tuning_table.entries.items():
        out[(key.op_kind, key.dtype, tuple(key.dims), t)] = (
            c.tile_m, c.tile_n, c.sm_footprint, c.efficiency_factor)
    return out


# ---- L4 coalescer (coalesce.py:56-131) ------------------------------------

def waste_of(op, member_flops, padded_dims):
    """coalesce.py:56-58 — 1 - sum(member) / (L * flops(padded))."""
    return 1.0 - sum(member_flops) / (len(member_flops) * op_flops(op, padded_dims))


def shape_groups(pending, budget):
    """coalesce.py:69-106 — greedy deterministic partition.

    Returns a list of (op, dtype, padded_dims, [members in admission order],
    waste). Sort key is (op, dtype, dims descending, kernel id); each
    unassigned kernel seeds a group and later kernels of the same op/dtype
    join iff the recomputed waste stays within the budget.
    """
    if not 0.0 <= budget < 1.0:
        raise ValueError(f"pad_budget must be in [0, 1), got {budget}")
    ordered = sorted(pending, key=lambda k: (k.op_kind, k.dtype,
                                             tuple(-d for d in k.dims), k.kernel_id))
    taken = set()
    groups = []
    for i, seed in enumerate(ordered):
        if seed.kernel_id in taken:
            continue
        taken.add(seed.kernel_id)
        members, fl, pad = [seed], [op_flops(seed.op_kind, seed.dims)], tuple(seed.dims)
        for cand in ordered[i + 1:]:
            if cand.kernel_id in taken or cand.op_kind != seed.op_kind \
                    or cand.dtype != seed.dtype:
                continue
            grown = tuple(a if a > b else b for a, b in zip(pad, cand.dims))
            cf = op_flops(cand.op_kind, cand.dims)
            if waste_of(seed.op_kind, fl + [cf], grown) <= budget:
                members.append(cand)
                fl.append(cf)
                pad = grown
                taken.add(cand.kernel_id)
        groups.append((seed.op_kind, seed.dtype, pad, members,
                       waste_of(seed.op_kind, fl, pad)))
    return groups


def superkernel_cost(profile, table, op, dtype, padded, batch, tenancy):
    """coalesce.py:109-123 — cost of a padded batch of `batch` members."""
    cfg = table_config(table, op, dtype, padded, tenancy)
    nb = batch * model_blocks(op, padded, cfg[0], cfg[1])
    f = batch * op_flops(op, padded)
    b = batch * op_bytes(op, padded, dtype)
    e = occupancy(profile, nb, cfg[3])
    return Cost(f, b, nb, e, roofline_ns(profile, f, b, e, path_of(dtype)))


# ---- portable RNG (rng.py:19-58) -------------------------------------------

_M64 = (1 << 64) - 1


class Mix64:
    """rng.py:19-42 — splitmix64; uniform() has 53 random mantissa bits."""

    def __init__(self, seed):
        self.s = seed & _M64

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & _M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self, lo=0.0, hi=1.0):
        return lo + (hi - lo) * ((self.next_u64() >> 11) * 2.0 ** -53)

    def expovariate(self, rate):
        return -math.log1p(-self.uniform()) / rate


def fnv1a64(data):
    """rng.py:45-50."""
    h = 0xCBF29CE484222325
    for byte in data:
        h = ((h ^ byte) * 0x100000001B3) & _M64
    return h


def derive_seed(seed, *labels):
    """rng.py:53-58."""
    h = seed & _M64
    for lab in labels:
        h = Mix64(h ^ fnv1a64(str(lab).encode())).next_u64()
    return h


# ---- L5 scheduler state machine (scheduler.py:39-471) ----------------------

Params = namedtuple("Params", "pad_budget max_delay_fraction straggler_threshold "
                              "eviction_window eviction_min_samples jitter_width "
                              "stagger_horizon duration_noise")
DEFAULT_PARAMS = Params(0.25, 0.5, 2.0, 32, 8, 0.15, 10_000, 0.0)   # scheduler.py:39-48


class Launch:
    """One dispatch record (scheduler.py:81-96)."""

    __slots__ = ("dispatch_id", "kernel_ids", "super_id", "stream_ids", "start",
                 "end", "sm_allocation", "context_id", "ctx_switch",
                 "useful_flops", "padded_flops", "predicted_duration",
                 "duration", "infeasible")

    def __init__(self, **kw):
        for name in self.__slots__:
            setattr(self, name, kw.get(name))

    def as_tuple(self):
        return tuple(getattr(self, n) for n in self.__slots__)


class OracleScheduler:
    """Restatement of `Scheduler` (scheduler.py:130-471), all five variants.

    State is kept in plain dicts; method names are the reference's public
    ones so the reference engine can drive it (`gpumux.engine.Scheduler` can
    be swapped for it in tests).
    """

    def __init__(self, profile, variant, params=DEFAULT_PARAMS, table=None,
                 rng_state=0, footprint=FOOTPRINT_MODEL):
        if variant not in ("fifo", "edf", "ooo", "time-mux", "space-mux"):
            raise ValueError(f"unknown policy {variant!r}")
        self.profile = profile
        self.variant = variant
        self.params = params
        self.table = table or {}
        self.rng = Mix64(rng_state)
        self.fp_base, self.fp_slope = footprint
        self.reqs = {}            # rid -> dict(request, remaining, evicted, done_at)
        self.owner = {}           # kid -> rid
        self.pos = {}             # kid -> index in request.kernels
        self.ready = {}           # kid -> kernel (insertion ordered)
        self.blocked = {}
        self.waiting_on = {}      # kid -> set of dep kids
        self.done = set()
        self.predicted = {}
        self.in_flight = {}
        self.free_sms = profile.sm_count
        self.last_ctx = None
        self.evicted_streams = set()
        self.rr_last = None
        self.withheld_sigs = set()
        self.seq = 0
        self.ratio_windows = {}

    # intake: scheduler.py:167-193
    def add_request(self, req):
        st = {"request": req, "remaining": {k.kernel_id for k in req.kernels},
              "evicted": False, "done_at": None}
        self.reqs[req.request_id] = st
        if req.stream_id in self.evicted_streams:
            st["evicted"] = True
            return False
        for i, k in enumerate(req.kernels):
            self.owner[k.kernel_id] = req.request_id
            self.pos[k.kernel_id] = i
            cfg = table_config(self.table, k.op_kind, k.dtype, k.dims, 1)
            self.predicted[k.kernel_id] = solo_cost(self.profile, k, cfg).duration
            if k.deps:
                self.blocked[k.kernel_id] = k
                self.waiting_on[k.kernel_id] = set(k.deps)
            else:
                self.ready[k.kernel_id] = k
        return True

    # scheduler.py:195-206
    def predicted_remaining(self, k):
        st = self.reqs[self.owner[k.kernel_id]]
        tail = st["request"].kernels[self.pos[k.kernel_id]:]
        return sum(self.predicted[s.kernel_id] for s in tail
                   if s.kernel_id not in self.done)

    def kernel_slack(self, k, now):
        return k.deadline - now - self.predicted_remaining(k)

    # completion: scheduler.py:210-235
    def complete(self, did, now, measured=None):
        """`measured`: an observed duration (ns) replacing the modeled one in the straggler
        ratio (the build's wall-clock engine; the reference always uses
        d.duration, i.e. measured=None)."""
        d = self.in_flight.pop(did)
        self.free_sms += d.sm_allocation
        finished = []
        ratio = (d.duration if measured is None else measured) / max(d.predicted_duration, 1)
        for kid in d.kernel_ids:
            self.done.add(kid)
            st = self.reqs[self.owner[kid]]
            st["remaining"].discard(kid)
            if not st["remaining"] and st["done_at"] is None:
                st["done_at"] = now
                finished.append((st["request"], now))
            for k in st["request"].kernels:
                w = self.waiting_on.get(k.kernel_id)
                if w is not None:
                    w.discard(kid)
                    if not w:
                        del self.waiting_on[k.kernel_id]
                        self.ready[k.kernel_id] = self.blocked.pop(k.kernel_id)
        for s in d.stream_ids:
            self.ratio_windows.setdefault(
                s, deque(maxlen=self.params.eviction_window)).append(ratio)
        return SimpleNamespace(dispatch=d, finished_requests=finished)

    # stragglers: scheduler.py:237-278
    def straggler_ratio(self, stream):
        w = self.ratio_windows.get(stream)
        if not w or len(w) < self.params.eviction_min_samples:
            return None
        srt = sorted(w)
        return srt[max(1, math.ceil(0.99 * len(srt))) - 1]

    def find_stragglers(self):
        out = []
        for s in sorted(self.ratio_windows):
            if s in self.evicted_streams:
                continue
            r = self.straggler_ratio(s)
            if r is not None and r > self.params.straggler_threshold:
                out.append(s)
        return out

    def evict_straggler(self, stream, now):
        self.evicted_streams.add(stream)
        cancelled = []
        for did, d in list(self.in_flight.items()):
            if set(d.stream_ids) == {stream}:
                cancelled.append(did)
                del self.in_flight[did]
                self.free_sms += d.sm_allocation
        gone = []
        for rid, st in self.reqs.items():
            if st["request"].stream_id != stream or st["done_at"] is not None:
                continue
            if not st["evicted"]:
                st["evicted"] = True
                gone.append(rid)
            for k in st["request"].kernels:
                self.ready.pop(k.kernel_id, None)
                self.blocked.pop(k.kernel_id, None)
                self.waiting_on.pop(k.kernel_id, None)
        return SimpleNamespace(stream_id=stream, time=now,
                               cancelled_dispatch_ids=tuple(cancelled),
                               evicted_request_ids=tuple(sorted(gone)))

    @property
    def requests(self):
        """rid -> view with `.evicted` (what the engine's metrics read)."""
        return {rid: SimpleNamespace(evicted=st["evicted"], completed_at=st["done_at"])
                for rid, st in self.reqs.items()}

    # helpers: scheduler.py:282-316, 331-333
    def _live_ready(self):
        return [k for k in self.ready.values() if k.stream_id not in self.evicted_streams]

    def _active(self):
        s = {k.stream_id for k in self.ready.values()}
        for d in self.in_flight.values():
            s.update(d.stream_ids)
        return sorted(s - self.evicted_streams)

    def _noise(self):
        w = self.params.duration_noise
        return 1.0 if w <= 0 else 1.0 + self.rng.uniform(-w, w)

    def _launch(self, kernels, now, duration, predicted, alloc, ctx,
                switch=False, super_id=None, useful=None, padded=None,
                infeasible=False):
        self.seq += 1
        start = now + (self.profile.context_switch_cost if switch else 0)
        if useful is None:
            useful = sum(op_flops(k.op_kind, k.dims) for k in kernels)
        d = Launch(dispatch_id=self.seq, kernel_ids=tuple(k.kernel_id for k in kernels),
                   super_id=super_id,
                   stream_ids=tuple(sorted({k.stream_id for k in kernels})),
                   start=start, end=start + duration, sm_allocation=alloc,
                   context_id=ctx, ctx_switch=switch, useful_flops=useful,
                   padded_flops=useful if padded is None else padded,
                   predicted_duration=predicted, duration=duration,
                   infeasible=infeasible)
        for k in kernels:
            self.ready.pop(k.kernel_id, None)
        self.in_flight[d.dispatch_id] = d
        self.free_sms -= alloc
        self.last_ctx = ctx
        return d

    def _solo_cfg(self, k):
        return table_config(self.table, k.op_kind, k.dtype, k.dims, 1)

    # policies: scheduler.py:320-454
    def step(self, now):
        v = self.variant
        if v in ("fifo", "edf"):
            return self._serial(now, v == "edf")
        if v == "time-mux":
            return self._round_robin(now)
        if v == "space-mux":
            return self._fair_share(now)
        return self._ooo(now)

    def _serial(self, now, by_deadline):
        live = self._live_ready()
        if self.in_flight or not live:
            return [], [], None
        key = (lambda k: (k.deadline, k.kernel_id)) if by_deadline else \
            (lambda k: (k.arrival, k.kernel_id))
        k = min(live, key=key)
        pred = solo_cost(self.profile, k, self._solo_cfg(k)).duration
        dur = math.ceil(pred * self._noise())
        return [self._launch([k], now, dur, pred, self.profile.sm_count, k.stream_id,
                             infeasible=self.kernel_slack(k, now) < 0)], [], None

    def _round_robin(self, now):
        if self.in_flight:
            return [], [], None
        live = self._live_ready()
        streams = sorted({k.stream_id for k in live})
        if not streams:
            return [], [], None
        if self.rr_last is None or self.rr_last >= streams[-1]:
            s = streams[0]
        else:
            s = next(x for x in streams if x > self.rr_last)
        self.rr_last = s
        k = min((k for k in live if k.stream_id == s),
                key=lambda k: (k.arrival, k.kernel_id))
        pred = solo_cost(self.profile, k, self._solo_cfg(k)).duration
        dur = math.ceil(pred * self._noise())
        switch = self.last_ctx is not None and self.last_ctx != s
        return [self._launch([k], now, dur, pred, self.profile.sm_count, s,
                             switch=switch,
                             infeasible=self.kernel_slack(k, now) < 0)], [], None

    def _slice_ns(self, k, tenants):
        """scheduler.py:372-391 — roofline on a fair 1/t slice, degraded."""
        cfg = self._solo_cfg(k)
        if tenants <= 1:
            return solo_cost(self.profile, k, cfg).duration
        share = 1.0 / tenants
        nb = model_blocks(k.op_kind, k.dims, cfg[0], cfg[1])
        cap = share * (self.profile.sm_count * self.profile.blocks_per_sm)
        occ = min(1.0, nb / cap)
        degr = self.fp_base + self.fp_slope * share
        base_peak = self.profile.peak_flops_dense if path_of(k.dtype) == "dense" \
            else self.profile.peak_flops_scalar
        peak = base_peak * share * occ * degr
        c = math.ceil(op_flops(k.op_kind, k.dims) / peak * 1e9)
        m = math.ceil(op_bytes(k.op_kind, k.dims, k.dtype)
                      / (self.profile.mem_bandwidth * share) * 1e9)
        return max(c, m)

    def _fair_share(self, now):
        active = self._active()
        t = len(active)
        if t == 0:
            return [], [], None
        alloc = max(1, self.profile.sm_count // t)
        busy = {s for d in self.in_flight.values() for s in d.stream_ids}
        width = self.params.jitter_width * (1 + t % 2) if t >= 2 else 0.0
        out = []
        for s in active:
            if s in busy:
                continue
            cands = [k for k in self._live_ready() if k.stream_id == s]
            if not cands or self.free_sms < alloc:
                continue
            k = min(cands, key=lambda k: (k.arrival, k.kernel_id))
            base = self._slice_ns(k, t)
            f = 1.0 + (self.rng.uniform(0.0, width) if width else 0.0)
            dur = math.ceil(base * f * self._noise())
            out.append(self._launch([k], now, dur, base, alloc, s,
                                    infeasible=self.kernel_slack(k, now) < 0))
        return out, [], None

    def _slo(self, k):
        return k.deadline - self.reqs[self.owner[k.kernel_id]]["request"].arrival

    def _ooo(self, now):
        """scheduler.py:414-471 — cluster, order, withhold-once, SM-gate."""
        live = self._live_ready()
        if not live:
            return [], [], None
        tenancy = max(1, len(self._active()))
        frac = self.params.max_delay_fraction
        ranked = []
        for g in shape_groups(live, self.params.pad_budget):
            members = g[3]
            sl = {k.kernel_id: self.kernel_slack(k, now) for k in members}
            late = any(v < 0 for v in sl.values())
            # third key: min over the dict's KEYS, i.e. the smallest kernel id
            ranked.append(((0 if late else 1, min(k.deadline for k in members),
                            min(sl)), g, sl, late))
        ranked.sort(key=lambda r: r[0])
        launched, held, wakeups = [], [], []
        for _, g, sl, late in ranked:
            op, dtype, pad, members, _w = g
            cost = superkernel_cost(self.profile, self.table, op, dtype, pad,
                                    len(members), tenancy)
            sig = frozenset(k.kernel_id for k in members)
            may_wait = (not late and cost.efficiency < 1.0 and
                        all(sl[k.kernel_id] >= frac * self._slo(k) for k in members))
            if may_wait and sig not in self.withheld_sigs:
                self.withheld_sigs.add(sig)
                held.append(tuple(k.kernel_id for k in members))
                horizon = now + self.params.stagger_horizon
                for k in members:
                    if k.deadline >= NO_DEADLINE:
                        continue
                    edge = int(k.deadline - self.predicted_remaining(k)
                               - frac * self._slo(k))
                    horizon = min(horizon, edge)
                wakeups.append(max(horizon, now + 1))
                continue
            alloc = min(self.profile.sm_count,
                        math.ceil(cost.block_count / self.profile.blocks_per_sm))
            if self.free_sms < alloc:
                continue
            dur = math.ceil(cost.duration * self._noise())
            useful = sum(op_flops(k.op_kind, k.dims) for k in members)
            launched.append(self._launch(
                list(members), now, dur, cost.duration, alloc, "jit",
                super_id="sk-" + "-".join(str(k.kernel_id) for k in members),
                useful=useful, padded=cost.flops, infeasible=late))
        return launched, held, (min(wakeups) if wakeups else None)
