"""Discrete-event harness: restatement of gpumux/engine.py (TEST INFRASTRUCTURE).

Used to check decision parity where the reference itself cannot be imported
(the GPU box) and to time the reference's decision path in `bench.py
--impl reference`. The scheduler under test is injected, so the same loop
drives `oracle.decisions.OracleScheduler` and the product's
`paper_1901_10008_b200.Scheduler`; byte-identical NDJSON traces and metrics
JSON are the parity criterion (reference tests/test_acceptance.py:150-162).

Citations are to /root/reference/pkg/src/gpumux/engine.py unless noted.
"""

from __future__ import annotations

import heapq
import json
import math
from collections import namedtuple

from .decisions import (DEFAULT_PARAMS, NO_DEADLINE, K, Mix64, OracleScheduler,
                        derive_seed)

ReqRec = namedtuple("ReqRec", "request_id stream_id kernels arrival deadline")

INTERACTIVE_SLO = (10_000_000, 10_000_000_000)   # kernels.py:28-29


def lower(library, name, batch=1):
    """kernels.py:174-199 — model -> linear dependency chain of prototypes."""
    if name not in library:
        raise KeyError(f"unknown model {name!r}")
    chain = []
    for i, p in enumerate(library[name]):
        op, dims, dtype = p["op_kind"], tuple(int(d) for d in p["dims"]), p["dtype"]
        if batch > 1:
            if op == "gemm":
                dims = (dims[0], dims[1] * batch, dims[2])
            elif op == "gemv":
                op, dims = "gemm", (dims[0], batch, dims[1])
            else:
                dims = (dims[0] * batch,)
        chain.append((op, dims, dtype, (i - 1,) if i else ()))
    return chain


def arrival_times(arrival, horizon, rng):
    """engine.py:160-177 — fixed schedule, Poisson, or periodic-burst Poisson."""
    kind = arrival["kind"]
    if kind == "fixed":
        return [int(t) for t in arrival.get("schedule", ()) if t <= horizon]
    per_ns = arrival["rate_per_s"] / 1e9
    factor = arrival.get("burst_factor", 4.0)
    period = arrival.get("burst_period_ns", 100_000_000)
    duty = arrival.get("burst_duty", 0.2)
    out, t = [], 0.0
    while True:
        rate = per_ns
        if kind == "burst" and (t % period) < duty * period:
            rate = per_ns * factor
        t += rng.expovariate(rate)
        if t > horizon:
            return out
        out.append(int(t))


def materialize(workload, library, seed=0):
    """engine.py:180-206 — requests with globally unique deterministic ids."""
    reqs, next_kid, next_rid = [], 0, 0
    for s in workload["streams"]:
        rng = Mix64(derive_seed(seed, "arrivals", s["stream_id"]))
        slo = NO_DEADLINE if s["slo_ns"] is None else int(s["slo_ns"])
        if s["slo_ns"] is not None and not INTERACTIVE_SLO[0] <= slo <= INTERACTIVE_SLO[1]:
            raise ValueError(f"interactive slo out of range: {slo}")
        protos = lower(library, s["model_name"], int(s.get("batch", 1)))
        for t in arrival_times(s["arrival"], int(workload["duration_ns"]), rng):
            deadline = min(t + slo, NO_DEADLINE)
            ks = tuple(K(next_kid + i, s["stream_id"], op, dims, dtype,
                         frozenset(next_kid + d for d in deps), t, deadline)
                       for i, (op, dims, dtype, deps) in enumerate(protos))
            next_kid += len(protos)
            reqs.append(ReqRec(next_rid, s["stream_id"], ks, t, deadline))
            next_rid += 1
    reqs.sort(key=lambda r: (r.arrival, r.request_id))
    return reqs


def nearest_rank(samples, p):
    """engine.py:209-217."""
    if not samples:
        raise ValueError("percentile of empty sample set")
    srt = sorted(samples)
    return srt[max(1, math.ceil(p * len(srt))) - 1]


def _summary(infos, useful, busy_sm_ns, window, span, profile):
    """engine.py:273-301."""
    done = [r for r in infos if r["status"] == "completed"]
    ev = [r for r in infos if r["status"] == "evicted"]
    pend = [r for r in infos if r["status"] == "pending"]
    lat = [r["latency"] for r in done]
    miss = sum(1 for r in done if not r["slo_met"]) + len(ev)
    att = len(done) + len(ev)
    busy_s = busy_sm_ns / profile.sm_count / 1e9
    return {
        "requests": len(infos), "completed": len(done), "evicted": len(ev),
        "pending": len(pend), "slo_misses": miss,
        "slo_attainment": (1.0 - miss / att) if att else 1.0,
        "throughput_rps": len(done) / (span / 1e9) if span else 0.0,
        "throughput_flops": useful / (span / 1e9) if span else 0.0,
        "latency_p50_ns": nearest_rank(lat, 0.5) if lat else None,
        "latency_p90_ns": nearest_rank(lat, 0.9) if lat else None,
        "latency_p99_ns": nearest_rank(lat, 0.99) if lat else None,
        "utilization": busy_sm_ns / (profile.sm_count * window) if window else 0.0,
        "flop_efficiency": useful / (profile.peak_flops_dense * busy_s) if busy_s else 0.0,
    }


def oracle_factory(profile, variant, params, table, rng_state):
    return OracleScheduler(profile, variant, params, table, rng_state)


def simulate(workload, library, profile, variant, seed=0, params=DEFAULT_PARAMS,
             table=None, factory=oracle_factory):
    """engine.py:304-446 — returns (trace_ndjson, metrics_json, timeline, sched).

    `factory(profile, variant, params, table, rng_state)` builds the scheduler
    under test; it must expose the reference Scheduler's public methods.
    """
    reqs = materialize(workload, library, seed)
    sched = factory(profile, variant, params, table,
                    derive_seed(seed, "jitter"))
    events, records, cancelled, finish = [], {}, {}, {}

    def rec(t, kind, **kw):
        events.append({"time": t, "kind": kind, **kw})

    heap = [(r.arrival, 1, r.request_id, r) for r in reqs]
    heapq.heapify(heap)
    wake_seq = 0
    while heap:
        now = heap[0][0]
        while heap and heap[0][0] == now:
            _, kind, eid, payload = heapq.heappop(heap)
            if kind == 0:
                if eid in cancelled:
                    continue
                info = sched.complete(eid, now)
                rec(now, "complete", dispatch_id=eid,
                    kernel_ids=list(info.dispatch.kernel_ids),
                    super_id=info.dispatch.super_id)
                for r, when in info.finished_requests:
                    finish[r.request_id] = when
            elif kind == 1:
                ok = sched.add_request(payload)
                rec(now, "arrival", request_id=payload.request_id,
                    stream_id=payload.stream_id)
                if not ok:
                    rec(now, "evict", stream_id=payload.stream_id,
                        request_ids=[payload.request_id], reason="stream-evicted")
        for s in sched.find_stragglers():
            ev = sched.evict_straggler(s, now)
            for did in ev.cancelled_dispatch_ids:
                cancelled[did] = now
            rec(now, "evict", stream_id=s, request_ids=list(ev.evicted_request_ids),
                reason="straggler")
        launched, held, wake = sched.step(now)
        for ids in held:
            rec(now, "withhold", kernel_ids=list(ids))
        for d in launched:
            if d.ctx_switch:
                rec(now, "context_switch", context_id=d.context_id)
            rec(d.start, "dispatch", dispatch_id=d.dispatch_id,
                kernel_ids=list(d.kernel_ids), super_id=d.super_id,
                sm_allocation=d.sm_allocation, context_id=d.context_id,
                end=d.end, infeasible=d.infeasible)
            records[d.dispatch_id] = d
            heapq.heappush(heap, (d.end, 0, d.dispatch_id, None))
        if wake is not None:
            wake_seq += 1
            heapq.heappush(heap, (wake, 2, wake_seq, None))

    timeline = []
    for did in sorted(records):
        d = records[did]
        end = d.end
        if did in cancelled:
            end = min(end, cancelled[did])
            if end <= d.start:
                continue
        timeline.append((d.start, end, d.sm_allocation,
                         d.super_id or ",".join(str(k) for k in d.kernel_ids),
                         d.context_id))

    horizon = int(workload["duration_ns"])
    sids = [s["stream_id"] for s in workload["streams"]]
    per_stream = {s: [] for s in sids}
    infos = []
    states = sched.requests
    for r in reqs:
        at = finish.get(r.request_id)
        st = states.get(r.request_id)
        if st is not None and st.evicted and at is None:
            status = "evicted"
        elif at is None or at > horizon:
            status = "pending"
        else:
            status = "completed"
        info = {"request_id": r.request_id, "stream_id": r.stream_id,
                "status": status,
                "latency": (at - r.arrival) if status == "completed" else None,
                "slo_met": status == "completed" and at <= r.deadline,
                "completed_at": at}
        infos.append(info)
        per_stream[r.stream_id].append(info)

    live = [d for d in records.values() if d.dispatch_id not in cancelled]
    flops_by, busy_by = {}, {s: 0 for s in sids}
    for d in live:
        share = d.useful_flops / len(d.stream_ids)
        for s in d.stream_ids:
            flops_by[s] = flops_by.get(s, 0) + share
            busy_by[s] = busy_by.get(s, 0) + \
                (d.end - d.start) * d.sm_allocation // len(d.stream_ids)
    done_at = [finish[i["request_id"]] for i in infos if i["status"] == "completed"]
    first = min((r.arrival for r in reqs), default=0)
    span = (max(done_at) - first) if done_at else 0
    window = max(horizon, max(done_at, default=0))
    g = _summary(infos, sum(d.useful_flops for d in live),
                 sum((d.end - d.start) * d.sm_allocation for d in live),
                 window, span, profile)
    streams = {s: _summary(per_stream[s], flops_by.get(s, 0), busy_by.get(s, 0),
                           window, span, profile) for s in sids}
    metrics = {"policy": variant, "profile": profile.name, "seed": seed,
               "duration_ns": horizon, "global": g, "streams": streams}
    trace = "".join(json.dumps(e, sort_keys=True) + "\n" for e in events)
    return (trace, json.dumps(metrics, indent=2, sort_keys=True) + "\n",
            timeline, sched)
