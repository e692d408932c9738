"""Sweep executor planner knobs on the C2 step: mean device time of the coalesced kernel
(CUDA graph of back-to-back launches, as bench.py's roofline leg) per setting.

usage: python tools/sweep_plan.py [name=v1,v2,... ...]   e.g. split_pct=40,60,100 max_split=8,32
"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import C2Bench, algorithmic_bytes, time_launch_only, time_resident  # noqa: E402

grid = {}
for arg in sys.argv[1:]:
    k, v = arg.split("=")
    grid[k] = [int(x) for x in v.split(",")]
if not grid:
    grid = {"split_pct": [60]}
b = C2Bench(replicas=int(os.environ.get("GMX_REPLICAS", "8")))
nbytes = algorithmic_bytes(b.shapes)
merge = grid.pop("merge", [1])
resident = grid.pop("resident", [0])
base_slots = [list(s) for s in b.slots]
for rs, mg, combo in itertools.product(resident, merge, itertools.product(*grid.values())):
    opts = dict(zip(grid.keys(), combo))
    for k, v in opts.items():
        b.ex.set_option(k, v)
    # merge=M: one launch covers M replicas' steps (per-step cost = time / M)
    b.slots = [sum((base_slots[(j + q) % len(base_slots)] for q in range(mg)), []) for j in range(len(base_slots))]
    t, plan = time_resident(b, 400)[::2] if rs else time_launch_only(b, 200)
    t /= mg
    opts["merge"] = mg
    opts["resident"] = rs
    if rs:
        import ctypes as C
        r = C.c_int64()
        b.ex._lib.gmx_exec_resident_relay_ns(b.ex._h, C.byref(r))
        opts["relay_us_per_step"] = round(r.value / 400 / 1e3, 3)
    print(json.dumps({"opts": opts, "kernel_us": round(t * 1e6, 3), "GBps": round(nbytes / t / 1e9, 1),
                      "n_items": plan["n_items"], "n_split_items": plan["n_split_items"],
                      "max_cta_cost": plan["max_cta_cost"], "mean_cta_cost": round(plan["mean_cta_cost"], 1)}),
          flush=True)
