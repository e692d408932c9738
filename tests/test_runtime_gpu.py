"""The native serving loop (gmx_runtime) against the oracle engine, on the GPU.

Lockstep mode keeps the reference's virtual clock, so every request's
completion time from the native loop must equal the one the restated
reference engine (oracle/sim.py, itself pinned to gpumux) computes for the
same workload — while the dispatched members really execute on the B200 and
their outputs match the numerics oracle.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import decisions as od  # noqa: E402
from oracle import numerics as on  # noqa: E402
from oracle import sim  # noqa: E402

from .conftest import load_golden  # noqa: E402


def _run_workload(workload, library, profile_name="b200", params=None, check_numerics=True, resident=False):
    import paper_1901_10008_b200 as gm
    from paper_1901_10008_b200.executor import Executor, OperandSet
    from paper_1901_10008_b200.runtime import Runtime

    prof_raw = load_golden("profiles.json")[profile_name]
    prof = gm.DeviceProfile(**prof_raw)
    pp = gm.PolicyParams(**(params or {}))
    ex = Executor()
    rt = Runtime(ex, prof, gm.SchedulerPolicy("ooo", pp), jitter_state=od.derive_seed(0, "jitter"))
    reqs = sim.materialize(workload, library, 0)
    ops = {}
    for r in reqs:
        slots = []
        for k in r.kernels:
            o = OperandSet(k.op_kind, k.dims, dtype=k.dtype, seed=k.kernel_id % 997)
            slots.append(o.register(ex))
            ops[k.kernel_id] = o
        rt.submit(gm.InferenceRequest(r.request_id, r.stream_id,
                                      tuple(gm.KernelSpec(k.kernel_id, k.stream_id, k.op_kind, k.dims, k.dtype,
                                                          k.deps, k.arrival, k.deadline) for k in r.kernels),
                                      r.arrival, gm.LatencyConstraint.batch()), slots)
    if resident:   # every scheduler step goes to ONE persistent launch's queue
        s = torch.cuda.current_stream()
        ex.resident_begin(s)
        try:
            stats = rt.run(stream=s)
        finally:
            ex.resident_end()
    else:
        stats = rt.run()
    torch.cuda.synchronize()
    got = dict(rt.drain_completions())
    # oracle: completion time per request from the restated reference engine
    _trace, _metrics, _tl, osched = sim.simulate(workload, library, od.Prof(**prof_raw), "ooo",
                                                 params=od.DEFAULT_PARAMS._replace(**(params or {})))
    want = {rid: st["done_at"] for rid, st in osched.reqs.items() if st["done_at"] is not None}
    assert got == want
    if check_numerics:
        for kid, o in ops.items():
            a = o.a.float().cpu().numpy()
            if o.op_kind == "gemm":
                ref = on.gemm(a, o.b.float().cpu().numpy(), o.dims[2])
            elif o.op_kind == "gemv":
                ref = on.gemv(a, o.b.float().cpu().numpy())
            else:
                ref = on.elementwise(a)
            got_c = o.c.float().cpu().numpy()
            tf32 = o.op_kind == "gemm" and o.a.dtype == torch.float32
            assert on.within(got_c, ref, o.c.dtype == torch.bfloat16, tf32), (kid, o.dims, on.rel_err(got_c, ref))
    return stats


@pytest.mark.parametrize("resident", [False, True])
def test_runtime_c2_matches_oracle_engine(resident):
    traces = load_golden("traces.json")
    wl = traces["workloads"]["c2_resnet50_16"]
    wl = dict(wl, streams=[dict(s, model_name="resnet50_like_fp16") for s in wl["streams"]])
    lib = dict(load_golden("models.json"))
    lib["resnet50_like_fp16"] = [dict(p, dtype="fp16") for p in lib["resnet50_like"]]
    stats = _run_workload(wl, lib, resident=resident)
    assert stats["completed_requests"] == 16 and stats["launches"] >= 1


@pytest.mark.parametrize("resident", [False, True])
def test_runtime_gemm16_fp32_tf32(resident):
    """The reference's bundled gemm16 workload (16 x gemm(64,3136,576) "fp32"): fp32 operands
    stay fp32 in HBM and run as tf32 UMMA; decisions vs the oracle engine, numerics vs float64 on
    the UNROUNDED fp32 operands (5e-3)."""
    traces = load_golden("traces.json")
    stats = _run_workload(traces["workloads"]["gemm16"], load_golden("models.json"), resident=resident)
    assert stats["completed_requests"] == 16


@pytest.mark.parametrize("resident", [False, True])
def test_runtime_resnet50_like_fp32_chains(resident):
    """models.json resnet50_like as the reference ships it (fp32, 13-kernel chains), 4 streams."""
    wl = {"duration_ns": 5_000_000, "streams": [
        {"stream_id": f"r{i}", "model_name": "resnet50_like", "slo_ns": 10_000_000,
         "arrival": {"kind": "fixed", "schedule": [0, 400_000 * (i + 1)]}} for i in range(4)]}
    stats = _run_workload(wl, load_golden("models.json"), resident=resident)
    assert stats["completed_requests"] == 8


@pytest.mark.parametrize("resident", [False, True])
def test_runtime_mixed_chains_match_oracle_engine(resident):
    lib = dict(load_golden("models.json"))
    wl = {"duration_ns": 2_000_000, "streams": [
        {"stream_id": f"m{i}", "model_name": m, "slo_ns": 10_000_000,
         "arrival": {"kind": "fixed", "schedule": [0, 150_000 * (i + 1)]}}
        for i, m in enumerate(["mixed_fp16", "tiny_chain", "resnet50_fc", "eltwise_fp32", "mixed_fp16"])]}
    stats = _run_workload(wl, lib, params={"stagger_horizon": 50_000}, resident=resident)
    assert stats["completed_requests"] == 10


@pytest.mark.parametrize("resident", [False, True])
def test_realtime_mode_replays_through_the_reference_scheduler(resident):
    """Wall-clock mode: arrivals at real times, completions from CUDA events. Replaying the
    logged (time, event) sequence through the oracle scheduler (pinned to gpumux) must
    reproduce every step's decisions: dispatch ids + members, withheld groups, wakeups."""
    import paper_1901_10008_b200 as gm
    from paper_1901_10008_b200.executor import Executor, OperandSet
    from paper_1901_10008_b200.runtime import Runtime

    prof_raw = load_golden("profiles.json")["b200"]
    ex = Executor()
    rt = Runtime(ex, gm.DeviceProfile(**prof_raw), gm.SchedulerPolicy("ooo"), mode="realtime")
    lib = dict(load_golden("models.json"))
    wl = {"duration_ns": 3_000_000, "streams": [
        {"stream_id": f"r{i:02d}", "model_name": ["mixed_fp16", "conv_fp16_a", "conv_fp16_b", "tiny_chain"][i % 4],
         "slo_ns": 10_000_000, "arrival": {"kind": "fixed", "schedule": [200_000 + 37_000 * i, 1_500_000 + 11_000 * i]}}
        for i in range(12)]}
    reqs = sim.materialize(wl, lib, 0)
    for r in reqs:
        slots = [OperandSet(k.op_kind, k.dims, dtype=k.dtype, seed=k.kernel_id).register(ex) for k in r.kernels]
        rt.submit(gm.InferenceRequest(r.request_id, r.stream_id,
                                      tuple(gm.KernelSpec(k.kernel_id, k.stream_id, k.op_kind, k.dims, k.dtype,
                                                          k.deps, k.arrival, k.deadline) for k in r.kernels),
                                      r.arrival, gm.LatencyConstraint(10_000_000)), slots)
    rt.set_origin_now()
    if resident:   # completions observed from the resident executor's host-mapped flags
        s = torch.cuda.current_stream()
        ex.resident_begin(s)
        try:
            stats = rt.run(until=2_000_000_000, stream=s)
        finally:
            ex.resident_end()
        torch.cuda.synchronize()
    else:
        stats = rt.run(until=2_000_000_000)
    assert stats["completed_requests"] == len(reqs)
    log = rt.replay_log()
    by_rid = {r.request_id: r for r in reqs}
    osched = od.OracleScheduler(od.Prof(**prof_raw), "ooo")
    i, steps = 0, 0
    while i < len(log):
        kind, t, a, kids = log[i]
        if kind == 0:
            osched.complete(a, t)
        elif kind == 1:
            osched.add_request(by_rid[a])
        elif kind == 5:
            launched, held, wake = osched.step(t)
            got_d, got_h, got_w = [], [], None
            i += 1
            while i < len(log) and log[i][0] in (2, 3, 4):
                k2, _t2, a2, kids2 = log[i]
                if k2 == 2:
                    got_d.append((a2, kids2))
                elif k2 == 3:
                    got_h.append(kids2)
                else:
                    got_w = None if a2 < 0 else a2
                i += 1
            assert got_d == [(d.dispatch_id, d.kernel_ids) for d in launched], t
            assert got_h == list(held) and got_w == wake, t
            steps += 1
            continue
        i += 1
    assert steps >= 4
