"""Generate the golden fixtures that pin the oracle and the product.

Runs the REAL reference (`gpumux` 0.1.0 from /root/reference/pkg/src) in the
build container — the reference does not exist on the GPU box, so its outputs
are committed here as small JSON fixtures:

  models.json     model library the workloads lower through (the bundled
                  reference library plus fp16 / elementwise chains used to
                  widen coverage; injected via gpumux.kernels._BUNDLED_LIBRARY)
  profiles.json   device profiles used (v100 preset + the b200 decision profile)
  costs.json      kernel_cost / form_superkernel / cluster_shapes outputs
  traces.json     engine.run() trace NDJSON + metrics JSON (sha256, plus the
                  full text for small cases) for bundled and random workloads
                  x all five policies x {v100, b200}

Usage:  python tests/golden/make_golden.py   (rewrites the fixtures in place)
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import gpumux  # noqa: E402
from gpumux import kernels as gk  # noqa: E402
from gpumux.coalesce import cluster_shapes, form_superkernel  # noqa: E402
from gpumux.device import load_profile  # noqa: E402
from gpumux.engine import WorkloadSpec, run  # noqa: E402
from gpumux.kernels import KernelSpec, kernel_cost, submit, LatencyConstraint  # noqa: E402
from gpumux.scheduler import PolicyParams, SchedulerPolicy  # noqa: E402
from gpumux.tuning import ClusterKey, TuningConfig, TuningTable, build_table  # noqa: E402

POLICIES = ("fifo", "edf", "ooo", "time-mux", "space-mux")

with open(os.path.join(REPO, "paper_1901_10008_b200", "data", "profiles.json")) as fh:
    B200 = json.load(fh)["profiles"]["b200"]

EXTRA_MODELS = {
    "mixed_fp16": [
        {"op_kind": "gemm", "dims": [256, 196, 512], "dtype": "fp16"},
        {"op_kind": "elementwise", "dims": [50176], "dtype": "fp16"},
        {"op_kind": "gemm", "dims": [64, 784, 256], "dtype": "fp16"},
        {"op_kind": "gemv", "dims": [1000, 2048], "dtype": "fp16"},
    ],
    "resnet50_fc": [{"op_kind": "gemv", "dims": [1000, 2048], "dtype": "fp32"}],
    "conv_fp16_a": [{"op_kind": "gemm", "dims": [64, 3136, 576], "dtype": "fp16"}],
    "conv_fp16_b": [{"op_kind": "gemm", "dims": [128, 784, 1152], "dtype": "fp16"}],
    "eltwise_fp32": [{"op_kind": "elementwise", "dims": [802816], "dtype": "fp32"},
                     {"op_kind": "elementwise", "dims": [200704], "dtype": "fp32"}],
    "tiny_chain": [{"op_kind": "gemm", "dims": [16, 16, 16], "dtype": "fp32"},
                   {"op_kind": "gemv", "dims": [33, 17], "dtype": "fp32"},
                   {"op_kind": "elementwise", "dims": [5], "dtype": "fp32"}],
}


def library():
    lib = dict(gk._BUNDLED_LIBRARY)
    lib.update(EXTRA_MODELS)
    return lib


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def bundled(name):
    from importlib import resources
    text = resources.files("gpumux.data.workloads").joinpath(name + ".json").read_text()
    return json.loads(text)


def random_workload(rng, idx):
    models = ["resnet50_like", "lstm_like", "gemv_1024", "gemm_64_3136_576",
              "resnet18_conv2_2", "mixed_fp16", "resnet50_fc", "conv_fp16_a",
              "conv_fp16_b", "eltwise_fp32", "tiny_chain", "resnet18_conv_chain"]
    n = rng.randint(1, 9)
    streams = []
    for i in range(n):
        kind = rng.choice(["fixed", "fixed", "poisson", "burst"])
        if kind == "fixed":
            arrival = {"kind": "fixed",
                       "schedule": sorted(rng.randint(0, 300_000) for _ in range(rng.randint(1, 4)))}
        elif kind == "poisson":
            arrival = {"kind": "poisson", "rate_per_s": rng.choice([2000.0, 5000.0, 20000.0])}
        else:
            arrival = {"kind": "burst", "rate_per_s": 3000.0, "burst_factor": 6.0,
                       "burst_period_ns": 2_000_000, "burst_duty": 0.3}
        streams.append({"stream_id": f"w{idx}s{i:02d}", "model_name": rng.choice(models),
                        "slo_ns": rng.choice([None, 10_000_000, 12_000_000, 50_000_000,
                                              200_000_000]),
                        "arrival": arrival, "batch": rng.choice([1, 1, 1, 2, 4])})
    return {"streams": streams, "duration_ns": rng.choice([1_000_000, 3_000_000, 10_000_000])}


PARAM_SETS = {
    "default": {},
    "stagger100us": {"stagger_horizon": 100_000},
    "eps0": {"pad_budget": 0.0},
    "eps05_delay09": {"pad_budget": 0.5, "max_delay_fraction": 0.9},
    "noisy_evict": {"duration_noise": 0.4, "straggler_threshold": 1.2,
                    "eviction_min_samples": 2, "eviction_window": 4},
    "noise_only": {"duration_noise": 0.25},
}


def main():
    lib = library()
    gk._BUNDLED_LIBRARY.clear()
    gk._BUNDLED_LIBRARY.update(lib)

    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
        json.dump(B200, fh)
        b200_path = fh.name
    profiles = {"v100": load_profile("v100"), "b200": load_profile(b200_path)}
    os.unlink(b200_path)

    # ---- costs / clusters -------------------------------------------------
    rng = random.Random(1901_10008)
    shapes = [("gemm", (64, 3136, 576)), ("gemm", (1024, 1024, 1024)), ("gemv", (1024, 1024)),
              ("gemv", (1000, 2048)), ("elementwise", (10_000,)), ("gemm", (8, 8, 8)),
              ("gemm", (4096, 4096, 4096)), ("elementwise", (1,))]
    for p in lib["resnet50_like"] + lib["resnet18_conv_chain"]:
        shapes.append((p["op_kind"], tuple(p["dims"])))
    for _ in range(60):
        op = rng.choice(["gemm", "gemv", "elementwise"])
        ar = {"gemm": 3, "gemv": 2, "elementwise": 1}[op]
        shapes.append((op, tuple(rng.randint(1, 5000) for _ in range(ar))))
    configs = [TuningConfig(64, 64), TuningConfig(128, 128), TuningConfig(16, 32, 0.5, 0.8),
               TuningConfig(128, 16, 1.0, 0.6)]
    cost_cases = []
    for pname, prof in profiles.items():
        for op, dims in shapes:
            for dtype in ("fp32", "fp16"):
                k = KernelSpec(0, "s", op, dims, dtype)
                for ci, cfg in enumerate(configs):
                    c = kernel_cost(k, cfg, prof)
                    cost_cases.append({"profile": pname, "op": op, "dims": list(dims),
                                       "dtype": dtype, "config": ci, "flops": c.flops,
                                       "bytes": c.bytes, "blocks": c.block_count,
                                       "eff": c.efficiency.hex(), "duration": c.duration})

    cluster_cases = []
    for case in range(150):
        n = rng.randint(1, 40)
        pending = []
        for i in range(n):
            op = rng.choice(["gemm", "gemm", "gemv", "elementwise"])
            ar = {"gemm": 3, "gemv": 2, "elementwise": 1}[op]
            if rng.random() < 0.5:
                dims = tuple(rng.randint(1, 600) for _ in range(ar))
            else:
                base = rng.choice([64, 128, 256, 512])
                dims = tuple(max(1, base + rng.randint(-40, 40)) for _ in range(ar))
            pending.append(submit(op, dims, rng.choice(["fp32", "fp16"]),
                                  LatencyConstraint(rng.choice([10_000_000, 50_000_000])),
                                  f"s{i % 7}", arrival=rng.randint(0, 1000),
                                  kernel_id=rng.randint(0, 10_000) * 64 + i))
        budget = rng.choice([0.0, 0.1, 0.25, 0.5, 0.9])
        tenancy = rng.randint(1, 20)
        out = []
        for cl in cluster_shapes(pending, budget):
            entry = {"ids": [k.kernel_id for k in cl.members], "padded": list(cl.padded_dims),
                     "waste": cl.waste.hex()}
            for pname, prof in profiles.items():
                sk = form_superkernel(cl, None, prof, tenancy)
                entry[pname] = [sk.flops, sk.bytes, sk.cost.block_count,
                                sk.cost.efficiency.hex(), sk.cost.duration, sk.super_id,
                                sk.earliest_deadline, sk.useful_flops]
            out.append(entry)
        cluster_cases.append({
            "pending": [[k.kernel_id, k.stream_id, k.op_kind, list(k.dims), k.dtype,
                         k.arrival, k.deadline] for k in pending],
            "budget": budget, "tenancy": tenancy, "clusters": out})

    # a tuning table for table-driven cases
    table_keys = [ClusterKey("gemm", "fp32", tuple(p["dims"])) for p in lib["resnet50_like"][:6]]
    table_keys += [ClusterKey("gemv", "fp32", (1024, 1024)),
                   ClusterKey("gemm", "fp32", (64, 3136, 576))]
    table = build_table(table_keys, 3, profiles["v100"], budget=256)

    with open(os.path.join(HERE, "costs.json"), "w") as fh:
        json.dump({"configs": [[c.tile_m, c.tile_n, c.sm_footprint, c.efficiency_factor]
                               for c in configs],
                   "cost_cases": cost_cases, "cluster_cases": cluster_cases},
                  fh, separators=(",", ":"))

    # ---- traces -----------------------------------------------------------
    workloads = {name: bundled(name) for name in ("gemm16", "gemv8", "adversarial")}
    workloads["c2_resnet50_16"] = {
        "streams": [{"stream_id": f"t{i:02d}", "model_name": "resnet50_like",
                     "slo_ns": 10_000_000, "arrival": {"kind": "fixed", "schedule": [0]}}
                    for i in range(16)],
        "duration_ns": 1_000_000_000}
    workloads["c4_poisson64"] = {
        "streams": [{"stream_id": f"p{i:02d}", "model_name": "resnet50_like",
                     "slo_ns": 10_000_000, "arrival": {"kind": "poisson", "rate_per_s": 100.0}}
                    for i in range(64)],
        "duration_ns": 20_000_000}
    workloads["c1_fc4"] = {
        "streams": [{"stream_id": f"f{i}", "model_name": "resnet50_fc",
                     "slo_ns": 10_000_000, "arrival": {"kind": "fixed", "schedule": [0]}}
                    for i in range(4)],
        "duration_ns": 1_000_000_000}
    for i in range(40):
        workloads[f"rand{i:02d}"] = random_workload(rng, i)

    cases = []
    for wname, wl in workloads.items():
        spec = WorkloadSpec.from_dict(wl)
        for pname, prof in profiles.items():
            param_names = ["default"]
            if wname.startswith("rand"):
                param_names.append(rng.choice(list(PARAM_SETS)))
            if wname in ("gemv8", "c2_resnet50_16"):
                param_names += ["stagger100us", "eps0"]
            for pn in param_names:
                for variant in POLICIES:
                    seed = rng.randint(0, 2**31) if wname.startswith("rand") else 0
                    use_table = (wname in ("c2_resnet50_16", "gemm16") and pname == "v100"
                                 and variant == "ooo")
                    for tbl in ([None, table] if use_table else [None]):
                        res = run(spec, prof, SchedulerPolicy(variant, PolicyParams(**PARAM_SETS[pn])),
                                  seed=seed, tuning_table=tbl)
                        tr = res.trace.to_ndjson()
                        mt = res.metrics.to_json()
                        entry = {"workload": wname, "profile": pname, "variant": variant,
                                 "params": pn, "seed": seed, "table": tbl is not None,
                                 "trace_sha256": sha(tr), "metrics_sha256": sha(mt),
                                 "n_events": len(res.trace.events)}
                        if len(tr) < 6000:
                            entry["trace"] = tr
                            entry["metrics"] = mt
                        cases.append(entry)

    with open(os.path.join(HERE, "traces.json"), "w") as fh:
        json.dump({"param_sets": PARAM_SETS, "workloads": workloads, "cases": cases,
                   "tuning_table": table.to_dict()}, fh, separators=(",", ":"))
    with open(os.path.join(HERE, "models.json"), "w") as fh:
        json.dump(lib, fh, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "profiles.json"), "w") as fh:
        json.dump({k: {f: getattr(v, f) for f in ("name", "sm_count", "blocks_per_sm",
                                                 "peak_flops_dense", "peak_flops_scalar",
                                                 "mem_bandwidth", "context_switch_cost")}
                   for k, v in profiles.items()}, fh, indent=1)
    print(f"costs: {len(cost_cases)} cost cases, {len(cluster_cases)} cluster cases; "
          f"traces: {len(cases)} cases over {len(workloads)} workloads")


if __name__ == "__main__":
    main()
