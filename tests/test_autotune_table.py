"""§8(f)3 hardware autotuner: the MEASURED TuningTable committed from a B200 run
(profiles/tuning_b200_measured.json, tools/autotune.py) is a valid reference-format table, and
the product scheduler's decisions with it stay bit-exact against the oracle (pinned to gpumux)."""

import json
import os
import sys

import pytest

import paper_1901_10008_b200 as gm
from oracle import sim

from .conftest import REF_SRC, load_golden, reference_available
from .test_core_parity import product_factory
from .test_oracle_golden import _prof, _table

TABLE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                     "tuning_b200_measured.json")


@pytest.fixture(scope="module")
def measured():
    with open(TABLE) as fh:
        return json.load(fh)


def test_measured_table_shape(measured):
    entries = measured["entries"]
    assert len(entries) == 13 and measured["provenance"]["tuner"].startswith("measured")
    for key, levels in entries.items():
        assert key.startswith("gemm:fp16:") and sorted(levels) == ["1", "2", "3", "4"]
        for cfg in levels.values():
            assert cfg["tile_m"] == 128 and cfg["tile_n"] in (64, 128)
            assert 0 < cfg["efficiency_factor"] <= 1 and 0 < cfg["sm_footprint"] <= 1
    table = gm.TuningTable.load(TABLE)
    key = gm.ClusterKey.from_string(next(iter(entries)))
    assert table.lookup(key, 9) == table.lookup(key, 4)   # tenancy clamps to the tuned maximum


@pytest.mark.parametrize("variant", ["ooo", "edf"])
def test_decisions_with_measured_table_match_oracle(measured, variant):
    """C2 (16 tenants, resnet50_like fp16) and a mixed-chain workload: product traces with the
    measured table are byte-identical to the oracle scheduler's."""
    models = dict(load_golden("models.json"))
    models["resnet50_like_fp16"] = [dict(p, dtype="fp16") for p in models["resnet50_like"]]
    prof = _prof(load_golden("profiles.json")["b200"])
    table = _table(measured)
    workloads = [
        {"duration_ns": 3_000_000, "streams": [
            {"stream_id": f"t{i:02d}", "model_name": "resnet50_like_fp16", "slo_ns": 10_000_000,
             "arrival": {"kind": "fixed", "schedule": [0, 1_000_000, 2_000_000]}} for i in range(16)]},
        {"duration_ns": 2_000_000, "streams": [
            {"stream_id": f"m{i}", "model_name": m, "slo_ns": 10_000_000,
             "arrival": {"kind": "poisson", "rate_per_s": 2000}}
            for i, m in enumerate(["resnet50_like_fp16", "mixed_fp16", "tiny_chain", "resnet50_like_fp16"])]},
    ]
    for wl in workloads:
        want = sim.simulate(wl, models, prof, variant, table=table)[:2]
        got = sim.simulate(wl, models, prof, variant, table=table, factory=product_factory)[:2]
        assert got == want


@pytest.mark.reference
@pytest.mark.skipif(not reference_available(), reason="reference tree not present")
def test_reference_loads_measured_table(measured):
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from gpumux.tuning import ClusterKey, TuningTable
    ref = TuningTable.load(TABLE)
    ours = gm.TuningTable.load(TABLE)
    for key_text, levels in measured["entries"].items():
        for t in levels:
            r = ref.lookup(ClusterKey.from_string(key_text), int(t))
            o = ours.lookup(gm.ClusterKey.from_string(key_text), int(t))
            assert (r.tile_m, r.tile_n, r.sm_footprint, r.efficiency_factor) == \
                (o.tile_m, o.tile_n, o.sm_footprint, o.efficiency_factor)
