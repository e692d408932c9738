"""Pin the oracle against the reference's own outputs (committed fixtures).

These run on CPU anywhere; the fixtures were produced by the real reference
(tests/golden/make_golden.py).
"""

import hashlib

import pytest

from oracle import decisions as od
from oracle import sim


def _prof(raw):
    return od.Prof(**raw)


def _params(param_sets, name):
    return od.DEFAULT_PARAMS._replace(**param_sets[name])


def _table(raw):
    out = {}
    for key, levels in raw.get("entries", {}).items():
        op, dtype, dims = key.split(":")
        dims = tuple(int(d) for d in dims.split("x"))
        for t, c in levels.items():
            out[(op, dtype, dims, int(t))] = (c["tile_m"], c["tile_n"], c["sm_footprint"],
                                              c["efficiency_factor"])
    return out


def test_cost_model_matches_reference(golden_costs, golden_profiles):
    cfgs = golden_costs["configs"]
    for c in golden_costs["cost_cases"]:
        prof = _prof(golden_profiles[c["profile"]])
        k = od.K(0, "s", c["op"], tuple(c["dims"]), c["dtype"], frozenset(), 0, od.NO_DEADLINE)
        got = od.solo_cost(prof, k, tuple(cfgs[c["config"]]))
        assert (got.flops, got.bytes, got.block_count, got.efficiency.hex(), got.duration) == \
            (c["flops"], c["bytes"], c["blocks"], c["eff"], c["duration"]), c


def test_clusters_and_superkernels_match_reference(golden_costs, golden_profiles):
    for case in golden_costs["cluster_cases"]:
        pend = [od.K(kid, s, op, tuple(d), dt, frozenset(), a, dl)
                for kid, s, op, d, dt, a, dl in case["pending"]]
        groups = od.shape_groups(pend, case["budget"])
        assert len(groups) == len(case["clusters"])
        for (op, dtype, pad, members, waste), want in zip(groups, case["clusters"]):
            assert [k.kernel_id for k in members] == want["ids"]
            assert list(pad) == want["padded"]
            assert waste.hex() == want["waste"]
            for pname in ("v100", "b200"):
                prof = _prof(golden_profiles[pname])
                c = od.superkernel_cost(prof, {}, op, dtype, pad, len(members), case["tenancy"])
                w = want[pname]
                assert [c.flops, c.bytes, c.block_count, c.efficiency.hex(), c.duration] == w[:5]


def _run_case(case, golden_traces, golden_models, golden_profiles, factory=sim.oracle_factory):
    wl = golden_traces["workloads"][case["workload"]]
    prof = _prof(golden_profiles[case["profile"]])
    params = _params(golden_traces["param_sets"], case["params"])
    table = _table(golden_traces["tuning_table"]) if case["table"] else None
    trace, metrics, _, _ = sim.simulate(wl, golden_models, prof, case["variant"],
                                        seed=case["seed"], params=params, table=table,
                                        factory=factory)
    return trace, metrics


def test_oracle_traces_match_reference(golden_traces, golden_models, golden_profiles):
    bad = []
    for case in golden_traces["cases"]:
        trace, metrics = _run_case(case, golden_traces, golden_models, golden_profiles)
        if "trace" in case and trace != case["trace"]:
            bad.append((case["workload"], case["profile"], case["variant"], "trace-text"))
        if hashlib.sha256(trace.encode()).hexdigest() != case["trace_sha256"]:
            bad.append((case["workload"], case["profile"], case["variant"], case["params"], "trace"))
        if hashlib.sha256(metrics.encode()).hexdigest() != case["metrics_sha256"]:
            bad.append((case["workload"], case["profile"], case["variant"], case["params"], "metrics"))
    assert not bad, bad[:10]


def test_rng_known_answers():
    # reference tests/test_rng.py pins seed-0 splitmix64 outputs
    r = od.Mix64(0)
    assert r.next_u64() == 0xE220A8397B1DCDAF
    assert r.next_u64() == 0x6E789E6AA1B965F4
