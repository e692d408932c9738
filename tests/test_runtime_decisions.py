"""The native serving loop (gmx_runtime) as a decisions-only engine (no executor) against the
oracle engine (oracle/sim.py, pinned to gpumux engine.run by the golden traces): every
request's completion time, every eviction (engine.py:345-351 straggler eviction with duration
noise), over all five policies and the golden parameter sets. Runs on CPU."""

import pytest

import paper_1901_10008_b200 as gm
from oracle import decisions as od
from oracle import sim

from .test_oracle_golden import _params, _prof, _table


def _native(wl, library, prof_raw, variant, params, table_raw, seed):
    from paper_1901_10008_b200.runtime import Runtime
    prof = gm.DeviceProfile(**prof_raw)
    pp = gm.PolicyParams(**params._asdict())
    tt = None
    if table_raw:
        tt = gm.TuningTable()
        for (op, dt, dims, t), c in _table(table_raw).items():
            tt.put(gm.ClusterKey(op, dt, dims), t, gm.TuningConfig(*c))
    rt = Runtime(None, prof, gm.SchedulerPolicy(variant, pp), tuning_table=tt,
                 jitter_state=od.derive_seed(seed, "jitter"))
    for r in sim.materialize(wl, library, seed):
        ks = tuple(gm.KernelSpec(k.kernel_id, k.stream_id, k.op_kind, k.dims, k.dtype, k.deps, k.arrival,
                                 k.deadline) for k in r.kernels)
        rt.submit(gm.InferenceRequest(r.request_id, r.stream_id, ks, r.arrival, gm.LatencyConstraint.batch()),
                  [0] * len(ks))
    stats = rt.run()
    return dict(rt.drain_completions(1 << 20)), stats


@pytest.mark.parametrize("param_set", ["noisy_evict", "noise_only", "stagger100us", "eps0"])
def test_native_engine_matches_oracle_engine(golden_traces, golden_models, golden_profiles, param_set):
    cases = [c for c in golden_traces["cases"] if c["params"] == param_set]
    assert cases
    evictions = 0
    for case in cases:
        wl = golden_traces["workloads"][case["workload"]]
        prof_raw = golden_profiles[case["profile"]]
        params = _params(golden_traces["param_sets"], case["params"])
        table_raw = golden_traces["tuning_table"] if case["table"] else None
        _tr, _m, _tl, osched = sim.simulate(wl, golden_models, _prof(prof_raw), case["variant"],
                                            seed=case["seed"], params=params,
                                            table=_table(table_raw) if table_raw else None)
        want = {rid: st["done_at"] for rid, st in osched.reqs.items() if st["done_at"] is not None}
        want_evicted = sum(1 for st in osched.reqs.values() if st.get("evicted") and st["done_at"] is None)
        got, stats = _native(wl, golden_models, prof_raw, case["variant"], params, table_raw, case["seed"])
        assert got == want, (case["workload"], case["variant"], case["profile"])
        assert stats["evicted_requests"] == want_evicted, (case["workload"], case["variant"])
        evictions += want_evicted
    if param_set == "noisy_evict":
        assert evictions > 0   # the straggler path really ran
