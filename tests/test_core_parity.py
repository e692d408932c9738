"""Decision parity of the native core against the reference's own outputs.

The product Scheduler (native C++ state machine behind the C ABI) is driven
by the oracle's restated event loop and must reproduce, byte for byte, the
NDJSON trace and metrics JSON the real reference produced for every golden
case (tests/golden/traces.json: bundled + C1/C2/C4-style + 40 random
workloads x 5 policies x {v100, b200} x parameter variants).
"""

import hashlib

import pytest

import paper_1901_10008_b200 as gm
from oracle import decisions as od
from oracle import sim

from .test_oracle_golden import _params, _prof, _table


def product_factory(profile, variant, params, table, rng_state):
    prof = gm.DeviceProfile(**profile._asdict())
    pp = gm.PolicyParams(**params._asdict())
    tt = None
    if table:
        tt = gm.TuningTable()
        for (op, dt, dims, t), c in table.items():
            tt.put(gm.ClusterKey(op, dt, dims), t, gm.TuningConfig(*c))
    rng = od.Mix64(rng_state)
    rng._state = rng.s
    return gm.Scheduler(prof, gm.SchedulerPolicy(variant, pp), tt, rng)


def test_product_traces_match_reference(golden_traces, golden_models, golden_profiles):
    bad = []
    for case in golden_traces["cases"]:
        wl = golden_traces["workloads"][case["workload"]]
        prof = _prof(golden_profiles[case["profile"]])
        params = _params(golden_traces["param_sets"], case["params"])
        table = _table(golden_traces["tuning_table"]) if case["table"] else None
        trace, metrics, _, _ = sim.simulate(wl, golden_models, prof, case["variant"],
                                            seed=case["seed"], params=params, table=table,
                                            factory=product_factory)
        if hashlib.sha256(trace.encode()).hexdigest() != case["trace_sha256"]:
            bad.append((case["workload"], case["profile"], case["variant"], case["params"], "trace"))
        elif hashlib.sha256(metrics.encode()).hexdigest() != case["metrics_sha256"]:
            bad.append((case["workload"], case["profile"], case["variant"], case["params"], "metrics"))
    assert not bad, f"{len(bad)} mismatches, e.g. {bad[:8]}"


def test_product_costs_match_reference(golden_costs, golden_profiles):
    cfgs = [gm.TuningConfig(*c) for c in golden_costs["configs"]]
    for c in golden_costs["cost_cases"]:
        prof = gm.DeviceProfile(**golden_profiles[c["profile"]])
        k = gm.KernelSpec(0, "s", c["op"], tuple(c["dims"]), c["dtype"])
        got = gm.kernel_cost(k, cfgs[c["config"]], prof)
        assert (got.flops, got.bytes, got.block_count, got.efficiency.hex(), got.duration) == \
            (c["flops"], c["bytes"], c["blocks"], c["eff"], c["duration"]), c


def test_product_clusters_match_reference(golden_costs, golden_profiles):
    profs = {p: gm.DeviceProfile(**golden_profiles[p]) for p in ("v100", "b200")}
    for case in golden_costs["cluster_cases"]:
        pend = [gm.KernelSpec(kid, s, op, tuple(d), dt, arrival=a, deadline=dl)
                for kid, s, op, d, dt, a, dl in case["pending"]]
        clusters = gm.cluster_shapes(pend, case["budget"])
        assert len(clusters) == len(case["clusters"])
        for cl, want in zip(clusters, case["clusters"]):
            assert [k.kernel_id for k in cl.members] == want["ids"]
            assert list(cl.padded_dims) == want["padded"]
            assert cl.waste.hex() == want["waste"]
            assert gm.pad_cost(cl).hex() == want["waste"]
            for pname, prof in profs.items():
                sk = gm.form_superkernel(cl, None, prof, case["tenancy"])
                assert [sk.flops, sk.bytes, sk.cost.block_count, sk.cost.efficiency.hex(),
                        sk.cost.duration, sk.super_id, sk.earliest_deadline,
                        sk.useful_flops] == want[pname]
